# A/B: compact back3d records + aligned vector walks (base) vs the previous HEAD (tune_old.so)
set -x
python -c "import __graft_entry__ as g; g.build()"
for c in c5 c4 c3; do
  python tools/time_iter.py $c 1
  CT_OSLALM_LIB=paper_1402_4381_b200/tune_old.so python tools/time_iter.py $c 1
done > gpurun_out/r30_ab.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "small or adjoint or accumulate or determinism_3d or full_size or two_streams or oslalm_3d or exchange_path_single_rank_3d or fista_3d or helical or zslab or degenerate or zcrop or whole_subset" > gpurun_out/r30_gputest.log 2>&1
tail -3 gpurun_out/r30_gputest.log
