# Debug build with device-side invariant checks (CT_DEBUG_CHECKS=1; compute-sanitizer is not
# available on the GPU pool): every kernel family on small cases plus the GPU parity and
# virtual-rank tests against it.  A failed check is a device assert (the run fails).
set -x
python -c "import __graft_entry__ as g; g.build()"
python -m paper_1402_4381_b200.build --out paper_1402_4381_b200/tune_debug.so -DCT_DEBUG_CHECKS=1 > /dev/null
export CT_OSLALM_LIB=paper_1402_4381_b200/tune_debug.so
python tools/sanitize_cases.py
python -m pytest tests/test_gpu_parity.py tests/test_virtual_ranks.py -x -q -k "not determinism"
