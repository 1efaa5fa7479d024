# call 7: fwd3d2 variants on OS-LALM iterations
set -x
export VARS="base: unpred:-DCT_FWD3D2_UNPRED=1 cps4m5:-DCT_FWD3D2_CPS4=1_-DCT_FWD3D2_MINB_HEL=5 cps4m6:-DCT_FWD3D2_CPS4=1 tc24:-DCT_FWD3D2_TC_HEL=24 tc28:-DCT_FWD3D2_TC_HEL=28"
export CFGS="c5 c4"
timeout 1800 bash tools/ab3d_iter.sh > gpurun_out/r7_ab.log 2>&1
