# A/B timing of 2D tuning variants (same box, same call)
python -c "import __graft_entry__ as g; g.build()"
timeout 400 python -m pytest tests -m gpu -x -q -k "fan or c1 or c2 or adjoint or determinism or small or exchange or bb or axis" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
for v in "base:" "abs:-DCT_VREL=0"; do
  name=${v%%:*}; flags=${v#*:}
  python -m paper_1402_4381_b200.build --out paper_1402_4381_b200/tune_$name.so $flags > /dev/null
done
for r in 1 2; do for name in base abs; do
  CT_OSLALM_LIB=paper_1402_4381_b200/tune_$name.so python tools/time_proj.py c2 30
done; done
