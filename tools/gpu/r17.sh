set -x
timeout 3000 python tools/parity_long.py c5 20 gpurun_out/parity_long_c5_z24.json 24 > gpurun_out/r17_c5.log 2>&1
timeout 3600 python tools/parity_long.py c4 30 gpurun_out/parity_long_c4_z64.json 64 > gpurun_out/r17_c4.log 2>&1
