# A/B of round-2 record compaction (back3d / fwd3d2) and the K3 class sums; old = 0be706f
set -x
python -c "import __graft_entry__ as g; g.build()"
python -c "from paper_1402_4381_b200 import ctlib; print(ctlib.lib().ct_build_info())" || true
B=paper_1402_4381_b200
python -m $B.build --out $B/tune_nv.so -DCT_BACK3D_VEC=0 > /dev/null
python -m $B.build --out $B/tune_ne.so -DCT_BACK3D_EAGER=0 > /dev/null
python -m $B.build --out $B/tune_fw1.so -DCT_FWD3D2_W1EAGER=1 > /dev/null
python -m $B.build --out $B/tune_k3o.so -DCT_K3_CLASS=0 > /dev/null
for c in c5 c4; do
  python tools/time_iter.py $c 1
  for v in old nv ne fw1 k3o; do CT_OSLALM_LIB=$B/tune_$v.so python tools/time_iter.py $c 1; done
done > gpurun_out/r31_ab.log 2>&1
