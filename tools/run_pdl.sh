python -c "import __graft_entry__ as g; g.build()"
timeout 400 python -m pytest tests -m gpu -x -q -k "fan or c1 or c2 or adjoint or determinism or small or exchange or bb" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
python -m paper_1402_4381_b200.build --out paper_1402_4381_b200/tune_nopdl.so -DCT_PDL=0 > /dev/null
for r in 1 2; do
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b_pdl.json 2>/dev/null
CT_OSLALM_LIB=paper_1402_4381_b200/tune_nopdl.so python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b_nopdl.json 2>/dev/null
python -c "
import json
for f in ('b_pdl','b_nopdl'):
    d=json.loads(open('gpurun_out/'+f+'.json').read().strip().splitlines()[-1]); print(f, '%.4e'%d['value'], d['ms_per_step'])"
done
F5="python bench.py --config c5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --iters 1"
$F5 > gpurun_out/plain_f5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"fwd3d_kernel|back3d_kernel|sqs_update3d" -s 80 -c 3 -o gpurun_out/full_c5b $F5 > gpurun_out/ncu_full5.log 2>&1
python tools/ncu_traffic.py gpurun_out/full_c5b.ncu-rep c5 gpurun_out/traffic5.json
