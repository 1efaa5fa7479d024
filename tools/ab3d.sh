# A/B of 3D variants on one box (same call)
python -c "import __graft_entry__ as g; g.build()"
for v in "base:" "F3:-DCT_FWD3D_MINB=3" "F5:-DCT_FWD3D_MINB=5" "B3:-DCT_BACK3D_MINB=3" "B5:-DCT_BACK3D_MINB=5"; do
  name=${v%%:*}; flags=${v#*:}
  python -m paper_1402_4381_b200.build --out paper_1402_4381_b200/tune_$name.so $flags > /dev/null
done
for c in c3 c5; do for name in base F3 F5 B3 B5; do
  CT_OSLALM_LIB=paper_1402_4381_b200/tune_$name.so python tools/time_proj.py $c 3
done; done
