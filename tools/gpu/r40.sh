# c4: view groups in the two-view rows path (base) vs off there (nr2v) vs off everywhere (ng); c5 check; full GPU suite
set -x
python -c "import __graft_entry__ as g; g.build()"
B=paper_1402_4381_b200
python -m $B.build --out $B/tune_nr2v.so -DCT_BACK3D_GROUP_R2V=0 > /dev/null
python -m $B.build --out $B/tune_ng.so -DCT_BACK3D_GROUP=0 > /dev/null
for c in c4 c5; do
  python tools/time_iter.py $c 1
  for v in nr2v ng; do CT_OSLALM_LIB=$B/tune_$v.so python tools/time_iter.py $c 1; done
done > gpurun_out/r40_ab.log 2>&1
grep -v "^+" gpurun_out/r40_ab.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r40_gputest.log 2>&1
tail -2 gpurun_out/r40_gputest.log
