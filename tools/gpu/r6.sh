# call 6: sanitizers on small cases; ncu source capture of the c5 step kernels; parity; bench
set -x
mkdir -p gpurun_out/san
python tools/sanitize_cases.py > gpurun_out/san/plain.log 2>&1
for t in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $t --print-limit 50 --target-processes all python tools/sanitize_cases.py > gpurun_out/san/$t.log 2>&1
  echo "rc=$?" >> gpurun_out/san/$t.log
done
python tools/prof_iter.py c5 2 > gpurun_out/r6_prof.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fwd3d2_kernel|back3d_kernel|sqs_update3d" -s 78 -c 3 -o gpurun_out/r6_full_c5 python tools/prof_iter.py c5 2 > gpurun_out/r6_ncu.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_virtual_ranks.py -x -q > gpurun_out/r6_gputest.log 2>&1
python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r6_bench_c5.json 2> gpurun_out/r6_bench_c5.err
