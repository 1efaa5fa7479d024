set -x
export VARS="base: ysplit:-DCT_FWD3D2_YSPLIT=1 nopref:-DCT_BACK3D_PREFETCH=0"
export CFGS="c5 c4 c3"
timeout 1800 bash tools/ab3d_iter.sh > gpurun_out/r11_ab.log 2>&1
