# call 3: fwd3d2 tile clipping A/B + projector parity
set -x
export VARS="base: noclip:-DCT_FWD3D2_CLIP=0 tc26:-DCT_FWD3D2_TC=26 tc32:-DCT_FWD3D2_TC=32 minb6:-DCT_FWD3D2_MINB=6 tc18:-DCT_FWD3D2_TC=18"
export CFGS="c5 c3 c4"
timeout 900 bash tools/ab3d.sh > gpurun_out/r3_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "small or full_size or adjoint or determinism or oslalm_3d or rows41 or fine or degenerate or zslab" > gpurun_out/r3_gputest.log 2>&1
