# call 8: device-side invariant checks (debug build) on every kernel family + parity tests
set -x
timeout 1500 bash tools/debug_checks.sh > gpurun_out/r8_debug_checks.log 2>&1
echo "rc=$?" >> gpurun_out/r8_debug_checks.log
