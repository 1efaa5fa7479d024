# A/B of 3D variants on one box (same call): VARS="name:-DFLAG=V ..." (base = default build)
python -c "import __graft_entry__ as g; g.build()"
VARS=${VARS:-"base: P0:-DCT_FWD3D_PAIR=0"}
CFGS=${CFGS:-"c3 c5"}
for v in $VARS; do
  name=${v%%:*}; flags=${v#*:}; flags=${flags//_-D/ -D}
  [ "$name" = base ] || python -m paper_1402_4381_b200.build --out paper_1402_4381_b200/tune_$name.so $flags > /dev/null
done
lib() { [ "$1" = base ] && echo paper_1402_4381_b200/libct_oslalm.so || echo paper_1402_4381_b200/tune_$1.so; }
for c in $CFGS; do for v in $VARS; do name=${v%%:*}
  CT_OSLALM_LIB=$(lib $name) python tools/time_proj.py $c 3
done; done
