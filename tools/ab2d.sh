# A/B timing of tuning variants (same box, same call): variants built in-tree as tuning .so files
python -c "import __graft_entry__ as g; g.build()"
for v in "F5B6:-DCT_FWD2D_MINB=5 -DCT_BACK2D_MINB=6" "F6B5:-DCT_FWD2D_MINB=6 -DCT_BACK2D_MINB=5" "F4B4:-DCT_FWD2D_MINB=4 -DCT_BACK2D_MINB=4"; do
  name=${v%%:*}; flags=${v#*:}
  python -m paper_1402_4381_b200.build --out paper_1402_4381_b200/tune_$name.so $flags > /dev/null
done
for r in 1 2; do for name in F5B6 F6B5 F4B4; do
  CT_OSLALM_LIB=paper_1402_4381_b200/tune_$name.so python tools/time_proj.py c2 30
done; done
