set -x
timeout 900 python -m pytest tests/test_virtual_ranks.py tests/test_gpu_parity.py -x -q > gpurun_out/r9_gputest.log 2>&1
