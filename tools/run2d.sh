python -c "import __graft_entry__ as g; g.build()"
timeout 400 python -m pytest tests -m gpu -x -q -k "fan or c1 or c2 or adjoint or determinism or small" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -4 gpurun_out/pytest_gpu.log
python tools/time_proj.py c2 20; python tools/time_proj.py c1 20
ncu --set full --import-source on --clock-control none -k regex:"fwd2d_tile|back2d" -c 2 -o gpurun_out/c2_2d_v4 python tools/prof_proj.py c2 1 > gpurun_out/ncu_c2.log 2>&1; echo ncu=$?
