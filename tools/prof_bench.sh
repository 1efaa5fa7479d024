# Profiles of the default bench workload (run under gpurun; writes gpurun_out/).
#   1) launch list (gpu__time_duration per kernel, cold/serialised): shares, not absolutes
#   2) one `--set full` capture of each step's kernels inside the timed iteration
set -x
CFG=${1:-c2}
python -c "import __graft_entry__ as g; g.build()"
python bench.py --config $CFG --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_prof_$CFG.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv \
    python bench.py --config $CFG --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_$CFG.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"fwd2d|fwd3d|back2d|back3d|sqs_update" \
    --launch-skip 100 -c 9 -o gpurun_out/full_$CFG python bench.py --config $CFG --steps 1 --warmup 1 --no-e2e \
    --no-cpu-baseline --iters 1 > gpurun_out/ncu_full_$CFG.log 2>&1
python tools/ncu_traffic.py gpurun_out/full_$CFG.ncu-rep $CFG gpurun_out/traffic.json
