set -x
export VARS="base: nointer:-DCT_FWD3D2_INTERIOR=0 inter_unpred:-DCT_FWD3D2_UNPRED=1"
export CFGS="c5 c4 c3"
timeout 1800 bash tools/ab3d_iter.sh > gpurun_out/r15_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "small or full_size or oslalm or adjoint or fine or rows41 or degenerate" > gpurun_out/r15_gputest.log 2>&1
