# A/B of 3D variants on one box (same call)
python -c "import __graft_entry__ as g; g.build()"
for v in "base:" "T32:-DCT_FWD3D_TC=32" "T24:-DCT_FWD3D_TC=24"; do
  name=${v%%:*}; flags=${v#*:}
  python -m paper_1402_4381_b200.build --out paper_1402_4381_b200/tune_$name.so $flags > /dev/null
done
for c in c3 c4 c5; do for name in base T32 T24; do
  CT_OSLALM_LIB=paper_1402_4381_b200/tune_$name.so python tools/time_proj.py $c 3
done; done
