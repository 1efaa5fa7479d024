set -x
timeout 3400 python tools/parity_long.py c4 20 gpurun_out/parity_long_c4_z64.json 64 > gpurun_out/r19_c4.log 2>&1
