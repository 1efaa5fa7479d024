set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_virtual_ranks.py -x -q > gpurun_out/r14_gputest.log 2>&1
python bench.py --steps 10 --warmup 3 --cpu-budget 5 > gpurun_out/r14_bench_c5.json 2> gpurun_out/r14_bench_c5.err
