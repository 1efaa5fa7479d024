# r43: back3d with view groups on — two-view rows for 64-row detectors (r2v64), 4 CTAs/SM (minb4), both
set -x
python -c "import __graft_entry__ as g; g.build()"
B=paper_1402_4381_b200
python -m $B.build --out $B/tune_r2v64.so -DCT_BACK3D_ROWS2V_64=1 > /dev/null
python -m $B.build --out $B/tune_minb4.so -DCT_BACK3D_MINB=4 > /dev/null
python -m $B.build --out $B/tune_both.so -DCT_BACK3D_ROWS2V_64=1 -DCT_BACK3D_MINB=4 > /dev/null
for c in c5 c3 c4; do
  python tools/time_iter.py $c 1
  for v in r2v64 minb4 both; do CT_OSLALM_LIB=$B/tune_$v.so python tools/time_iter.py $c 1; done
  python tools/time_iter.py $c 1
done > gpurun_out/r43_ab.log 2>&1
rm -f $B/tune_*.so
grep -v "^+" gpurun_out/r43_ab.log
