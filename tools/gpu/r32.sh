# A/B: polynomial l_theta (lp), y-split forward (ys) vs base (K3 class sums) and 0be706f (old)
set -x
python -c "import __graft_entry__ as g; g.build()"
B=paper_1402_4381_b200
python -m $B.build --out $B/tune_lp.so -DCT_LPOLY=1 > /dev/null
python -m $B.build --out $B/tune_ys.so -DCT_FWD3D2_YSPLIT=1 > /dev/null
for c in c5 c4 c3; do
  python tools/time_iter.py $c 1
  for v in lp ys old; do CT_OSLALM_LIB=$B/tune_$v.so python tools/time_iter.py $c 1; done
done > gpurun_out/r32_ab.log 2>&1
for v in base ys; do
  L=$B/libct_oslalm.so; [ $v = ys ] && L=$B/tune_ys.so
  CT_OSLALM_LIB=$L ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:fwd3d2 -s 60 -c 4 --csv python tools/prof_iter.py c5 2 > gpurun_out/r32_dram_$v.csv 2> gpurun_out/r32_dram_$v.err
done
CT_OSLALM_LIB=$B/tune_lp.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "adjoint or fwd_back_small or full_size or oslalm_3d or whole_subset or determinism_3d or zcrop" > gpurun_out/r32_gputest_lp.log 2>&1
tail -2 gpurun_out/r32_gputest_lp.log
