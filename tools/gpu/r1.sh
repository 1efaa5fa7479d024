set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r1_gpu.txt
python bench.py --steps 5 --warmup 2 --cpu-budget 5 > gpurun_out/r1_bench_c5.json 2> gpurun_out/r1_bench_c5.err
python tools/prof_proj.py c5 1 > gpurun_out/r1_prof.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fwd3d2_kernel|back3d_kernel" -c 2 -o gpurun_out/r1_full_c5 python tools/prof_proj.py c5 1 > gpurun_out/r1_ncu.log 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/r1_gputest.log 2>&1
tail -3 gpurun_out/r1_gputest.log
