# call 4: fwd3d2 tile-size / occupancy A/B; full-size parity tests (timed)
set -x
export VARS="base: tc32:-DCT_FWD3D2_TC=32 tc40:-DCT_FWD3D2_TC=40 tc48:-DCT_FWD3D2_TC=48 tc32m6:-DCT_FWD3D2_TC=32_-DCT_FWD3D2_MINB=6 tc40m6:-DCT_FWD3D2_TC=40_-DCT_FWD3D2_MINB=6 tc26m6:-DCT_FWD3D2_TC=26_-DCT_FWD3D2_MINB=6"
export CFGS="c5 c4 c3"
timeout 900 bash tools/ab3d.sh > gpurun_out/r4_ab.log 2>&1
nproc > gpurun_out/r4_nproc.txt; lscpu | head -20 >> gpurun_out/r4_nproc.txt
timeout 1800 python -m pytest tests/test_gpu_fullsize.py -x -q --durations=20 > gpurun_out/r4_fullsize.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k reg_grad > gpurun_out/r4_reg.log 2>&1
