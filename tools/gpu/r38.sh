# A/B: register-accumulated view groups in back3d (base: 8 views) vs off (ng), 4 (g4), 16 (g16)
set -x
python -c "import __graft_entry__ as g; g.build()"
B=paper_1402_4381_b200
python -m $B.build --out $B/tune_ng.so -DCT_BACK3D_GROUP=0 > /dev/null
python -m $B.build --out $B/tune_g4.so -DCT_BACK3D_GROUP=4 > /dev/null
python -m $B.build --out $B/tune_g16.so -DCT_BACK3D_GROUP=16 > /dev/null
for c in c5 c3; do
  python tools/time_iter.py $c 1
  for v in ng g4 g16; do CT_OSLALM_LIB=$B/tune_$v.so python tools/time_iter.py $c 1; done
done > gpurun_out/r38_ab.log 2>&1
grep -v "^+" gpurun_out/r38_ab.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "fwd_back_small or adjoint or oslalm_3d or determinism_3d or zcrop or whole_subset or exchange_path_single_rank_3d or fista_3d or sqs_denom or degenerate" > gpurun_out/r38_gputest.log 2>&1
tail -2 gpurun_out/r38_gputest.log
