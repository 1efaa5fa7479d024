# Round profile set (run under gpurun; writes gpurun_out/).  See profiles/README.md.
set -x
python -c "import __graft_entry__ as g; g.build()"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
# the driver's bench commands (c5 default: one step = one OS-LALM iteration)
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_ref.err
for c in c2 c3 c4; do python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
# launch list of bench steps (cold, serialised: compare shares): 2 timed steps of c5
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ct::|fwd3d|back3d|sqs_update|extent|xi_|mask_|init_scalars|zero_offmask|count_vv|l2_read" -c 5000 --csv --log-file gpurun_out/launches_c5.csv $B > gpurun_out/ncu_launch.log 2>&1
python tools/launch_summary.py gpurun_out/launches_c5.csv > gpurun_out/launches_c5_summary.txt
# one full capture of each c5 step kernel inside an OS-LALM iteration + DRAM traffic
python tools/prof_iter.py c5 2 > gpurun_out/prof_iter.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"fwd3d2_kernel|back3d_kernel|sqs_update3d" -s 78 -c 3 -o gpurun_out/full_c5 python tools/prof_iter.py c5 2 > gpurun_out/ncu_full5.log 2>&1
python tools/ncu_traffic.py gpurun_out/full_c5.ncu-rep c5 gpurun_out/traffic.json
python tools/ncu_summary.py gpurun_out/full_c5.ncu-rep > gpurun_out/ncu_full_c5_iter_kernels.txt
python -m pytest tests -m gpu -q --durations=15 > gpurun_out/gputest.log 2>&1
