# A/B: software-pipelined K3 planes (base) vs CT_K3_PIPE=0 (np); back3d 4 CTAs/SM (b4)
set -x
python -c "import __graft_entry__ as g; g.build()"
B=paper_1402_4381_b200
python -m $B.build --out $B/tune_np.so -DCT_K3_PIPE=0 > /dev/null
python -m $B.build --out $B/tune_b4.so -DCT_BACK3D_MINB=4 > /dev/null
for c in c5 c4 c3; do
  python tools/time_iter.py $c 1
  for v in np b4; do CT_OSLALM_LIB=$B/tune_$v.so python tools/time_iter.py $c 1; done
done > gpurun_out/r34_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "oslalm_3d or determinism_3d or exchange_path_single_rank_3d or fista_3d or zslab or zcrop or c3_full" > gpurun_out/r34_gputest.log 2>&1
tail -2 gpurun_out/r34_gputest.log
