# A/B: back3d view groups with the unions in the table (base) vs in registers (greg) vs off (ng); 16 (g16)
set -x
python -c "import __graft_entry__ as g; g.build()"
B=paper_1402_4381_b200
python -m $B.build --out $B/tune_greg.so -DCT_BACK3D_GROUP_SMEM=0 > /dev/null
python -m $B.build --out $B/tune_ng.so -DCT_BACK3D_GROUP=0 > /dev/null
python -m $B.build --out $B/tune_g16.so -DCT_BACK3D_GROUP=16 > /dev/null
python -m $B.build --out $B/tune_g32.so -DCT_BACK3D_GROUP=32 > /dev/null
for c in c5 c3; do
  python tools/time_iter.py $c 1
  for v in greg ng g16 g32; do CT_OSLALM_LIB=$B/tune_$v.so python tools/time_iter.py $c 1; done
  python tools/time_iter.py $c 1
done > gpurun_out/r39_ab.log 2>&1
grep -v "^+" gpurun_out/r39_ab.log
