set -x
export VARS="base: no2v:-DCT_BACK3D_ROWS2V=0"
export CFGS="c5 c3"
timeout 900 bash tools/ab3d_iter.sh > gpurun_out/r20_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_virtual_ranks.py -x -q > gpurun_out/r20_gputest.log 2>&1
