# round-2 call 2: virtual-rank tests, fwd3d2 A/B, gpu tests, short c5 bench
set -x
export VARS="base: noKS:-DCT_FWD3D2_KS=0 noACC4:-DCT_FWD3D2_ACC4=0 old:-DCT_FWD3D2_KS=0_-DCT_FWD3D2_ACC4=0"
export CFGS="c3 c5 c4"
timeout 900 bash tools/ab3d.sh > gpurun_out/r2_ab.log 2>&1
timeout 900 python -m pytest tests/test_virtual_ranks.py -x -q > gpurun_out/r2_virtual.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputest.log 2>&1
python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench_c5.json 2> gpurun_out/r2_bench_c5.err
