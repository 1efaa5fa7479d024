set -x
export VARS="base: nw2m12:-DCT_FWD3D2_NW=2_-DCT_FWD3D2_MINB_HEL=12 nw8m3:-DCT_FWD3D2_NW=8_-DCT_FWD3D2_MINB_HEL=3 tc20m7:-DCT_FWD3D2_TC_HEL=20_-DCT_FWD3D2_MINB_HEL=7"
export CFGS="c5 c4"
timeout 1800 bash tools/ab3d_iter.sh > gpurun_out/r12_ab.log 2>&1
timeout 3600 python tools/parity_long.py c3 20 gpurun_out/parity_long_c3.json > gpurun_out/r12_parity_long.log 2>&1
