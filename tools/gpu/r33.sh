# geometry-gated polynomial l_theta (default) vs 0be706f (old); full GPU suite
set -x
python -c "import __graft_entry__ as g; g.build()"
B=paper_1402_4381_b200
for c in c5 c4 c3; do
  python tools/time_iter.py $c 1
  CT_OSLALM_LIB=$B/tune_old.so python tools/time_iter.py $c 1
done > gpurun_out/r33_ab.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r33_gputest.log 2>&1
tail -2 gpurun_out/r33_gputest.log
