# r44: two-view rows phase on for 64-row detectors (with view groups): bench lines and the full GPU suite
set -x
python -c "import __graft_entry__ as g; g.build()"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
for c in c3 c4; do python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/gputest.log 2>&1
tail -3 gpurun_out/gputest.log
