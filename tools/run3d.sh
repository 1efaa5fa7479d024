python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests -m gpu -x -q -k "helical or axial or c3 or c4 or c5 or exchange or determinism or 3d" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -4 gpurun_out/pytest_gpu.log
for c in c3 c4 c5; do python tools/time_proj.py $c 3; done
