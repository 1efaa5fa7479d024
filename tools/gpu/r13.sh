set -x
export VARS="base: noblk:-DCT_BACK3D_BLOCKED=0 tc16nw8m4:-DCT_FWD3D2_TC_HEL=16_-DCT_FWD3D2_MINB_HEL=4 tc22nw8m3:-DCT_FWD3D2_TC_HEL=22"
export CFGS="c5 c4 c3"
timeout 1800 bash tools/ab3d_iter.sh > gpurun_out/r13_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_virtual_ranks.py -x -q > gpurun_out/r13_gputest.log 2>&1
