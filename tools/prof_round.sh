# Round profile set (run under gpurun; writes gpurun_out/).  See profiles/README.md.
set -x
python -c "import __graft_entry__ as g; g.build()"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 9000 -c 3000 --csv --log-file gpurun_out/launches_c2.csv $B > gpurun_out/ncu_launch.log 2>&1
F="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --iters 1"
$F > gpurun_out/plain_f.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"fwd2d_tile|fwd2d_finalize|back2d|sqs_update" -s 120 -c 4 -o gpurun_out/full_c2 $F > gpurun_out/ncu_full.log 2>&1
python tools/ncu_traffic.py gpurun_out/full_c2.ncu-rep c2 gpurun_out/traffic.json
for c in c3 c4 c5; do python bench.py --config $c --iters 2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_c2_reference.json 2> gpurun_out/bench_ref.err
# c5: one full capture of each step kernel inside an OS-LALM iteration + traffic (76 matching
# launches per step: setup fwd/back, init fwd/back, 24 x (sqs, fwd, back); -s 98 lands in step 2)
F5="python bench.py --config c5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --iters 1"
$F5 > gpurun_out/plain_f5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"fwd3d_kernel|fwd3d2_kernel|back3d_kernel|sqs_update3d" -s 98 -c 3 -o gpurun_out/full_c5 $F5 > gpurun_out/ncu_full5.log 2>&1
python tools/ncu_traffic.py gpurun_out/full_c5.ncu-rep c5 gpurun_out/traffic.json
