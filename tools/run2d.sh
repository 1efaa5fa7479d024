python -c "import __graft_entry__ as g; g.build()"
timeout 400 python -m pytest tests -m gpu -x -q -k "fan or c1 or c2 or adjoint or determinism or small" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -4 gpurun_out/pytest_gpu.log
python tools/time_proj.py c2 20; python tools/time_proj.py c1 20
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_quick.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_quick.log').read().strip().splitlines()[-1]); print('bench', d['value'], d['roofline']['frac'], {k:v['ms_total']/v['launches'] for k,v in d['kernel_ms'].items()})"
