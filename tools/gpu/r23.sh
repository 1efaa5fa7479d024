set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_virtual_ranks.py -x -q > gpurun_out/r23_gputest.log 2>&1
for c in c5 c4 c3 c2; do timeout 300 python tools/time_iter.py $c 1; done > gpurun_out/r23_time.log 2>&1
