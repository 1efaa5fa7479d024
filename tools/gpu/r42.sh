# r42: the multi-rank suite (virtual ranks; windowed z-slab exchange) and the z-slab parity cases at 5e7ad93+
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests/test_virtual_ranks.py tests/test_gpu_parity.py -k "zslab or virtual or band or row_slab" -q -m gpu --durations=10 > gpurun_out/r42_vr.log 2>&1
tail -15 gpurun_out/r42_vr.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r42_smoke.log 2>&1; tail -2 gpurun_out/r42_smoke.log
