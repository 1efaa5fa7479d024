set -x
python -c "import __graft_entry__ as g; g.build()"
python -m paper_1402_4381_b200.build --out paper_1402_4381_b200/tune_nb.so -DCT_FWD3D2_BOTH=0 > /dev/null
for c in c5 c4 c3; do
  python tools/time_iter.py $c 1
  CT_OSLALM_LIB=paper_1402_4381_b200/tune_nb.so python tools/time_iter.py $c 1
done > gpurun_out/r25_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_virtual_ranks.py -x -q > gpurun_out/r25_gputest.log 2>&1
