# call 5: back3d two-view walks A/B; fwd3d2 per-kind tiles; projector parity; bench
set -x
export VARS="base: pairm5:-DCT_BACK3D_MINB=5 nopair:-DCT_BACK3D_PAIR=0"
export CFGS="c5 c4 c3"
timeout 900 bash tools/ab3d.sh > gpurun_out/r5_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_virtual_ranks.py -x -q > gpurun_out/r5_gputest.log 2>&1
python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r5_bench_c5.json 2> gpurun_out/r5_bench_c5.err
