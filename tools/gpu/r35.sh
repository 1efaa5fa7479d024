# A/B on the current code: fwd3d2 without the unconditional first-4-channel updates (acc4o),
# 24-channel helical tiles (tc24), back3d two-view rows phase on the 64-row detector (r2v)
set -x
python -c "import __graft_entry__ as g; g.build()"
B=paper_1402_4381_b200
python -m $B.build --out $B/tune_acc4o.so -DCT_FWD3D2_ACC4=0 > /dev/null
python -m $B.build --out $B/tune_tc24.so -DCT_FWD3D2_TC_HEL=24 > /dev/null
python -m $B.build --out $B/tune_r2v.so -DCT_BACK3D_ROWS2V_64=1 > /dev/null
for c in c5 c4; do
  python tools/time_iter.py $c 1
  for v in acc4o tc24 r2v; do CT_OSLALM_LIB=$B/tune_$v.so python tools/time_iter.py $c 1; done
  python tools/time_iter.py $c 1
done > gpurun_out/r35_ab.log 2>&1
