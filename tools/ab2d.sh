# A/B timing of 2D tuning variants (same box, same call)
python -c "import __graft_entry__ as g; g.build()"
for v in "base:" "P:-DCT_BACK2D_PAIR=1" "P5:-DCT_BACK2D_PAIR=1 -DCT_BACK2D_MINB=4"; do
  name=${v%%:*}; flags=${v#*:}
  python -m paper_1402_4381_b200.build --out paper_1402_4381_b200/tune_$name.so $flags > /dev/null
done
for r in 1 2; do for name in base P P5; do
  CT_OSLALM_LIB=paper_1402_4381_b200/tune_$name.so python tools/time_proj.py c2 30
done; done
