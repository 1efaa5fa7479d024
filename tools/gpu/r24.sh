set -x
python -c "import __graft_entry__ as g; g.build()"
python -m paper_1402_4381_b200.build --out paper_1402_4381_b200/tune_xh.so -DCT_FWD3D2_XHINT=1 > /dev/null
for c in c5 c4 c3; do
  python tools/time_iter.py $c 1
  CT_OSLALM_LIB=paper_1402_4381_b200/tune_xh.so python tools/time_iter.py $c 1
  CT_L2_PERSIST_MB=80 CT_OSLALM_LIB=paper_1402_4381_b200/tune_xh.so python tools/time_iter.py $c 1
  CT_L2_PERSIST_MB=80 python tools/time_iter.py $c 1
done > gpurun_out/r24_ab.log 2>&1
