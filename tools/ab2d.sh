# A/B timing of 2D tuning variants (same box, same call)
python -c "import __graft_entry__ as g; g.build()"
for v in "base:" "V11:-DCT_F2VC=11" "V14:-DCT_F2VC=14" "V6:-DCT_F2VC=6" "B8:-DCT_B2VB=8" "B32:-DCT_B2VB=32"; do
  name=${v%%:*}; flags=${v#*:}
  python -m paper_1402_4381_b200.build --out paper_1402_4381_b200/tune_$name.so $flags > /dev/null
done
for r in 1 2; do for name in base V11 V14 V6 B8 B32; do
  CT_OSLALM_LIB=paper_1402_4381_b200/tune_$name.so python tools/time_proj.py c2 30
done; done
