# 20-iteration builder-run parity at HEAD kernels (polynomial l_theta, K3 class sums): c5 central 24 slices
set -x
python -c "import __graft_entry__ as g; g.build()"
python -c "from paper_1402_4381_b200 import ctlib; print(ctlib._lib().ct_build_info() if hasattr(ctlib,'_lib') else '')" || true
timeout 2700 python tools/parity_long.py c5 20 gpurun_out/parity_long_c5_z24_20iters.json 24 > gpurun_out/r36_parity.log 2>&1
tail -3 gpurun_out/r36_parity.log
