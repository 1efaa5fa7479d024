# r41: c4 A/B of view groups in the two-view rows path (base vs nr2v vs ng), then the round profile set at HEAD
set -x
python -c "import __graft_entry__ as g; g.build()"
B=paper_1402_4381_b200
python -m $B.build --out $B/tune_nr2v.so -DCT_BACK3D_GROUP_R2V=0 > /dev/null
python -m $B.build --out $B/tune_ng.so -DCT_BACK3D_GROUP=0 > /dev/null
for c in c4; do
  python tools/time_iter.py $c 1
  for v in nr2v ng; do CT_OSLALM_LIB=$B/tune_$v.so python tools/time_iter.py $c 1; done
  python tools/time_iter.py $c 1
done > gpurun_out/r41_ab.log 2>&1
rm -f $B/tune_*.so
bash tools/prof_round.sh
