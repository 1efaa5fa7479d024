# A/B of build variants on OS-LALM iterations (tools/time_iter.py): VARS="name:-DFLAG=V[_-DFLAG2=V2] ..."
python -c "import __graft_entry__ as g; g.build()"
VARS=${VARS:-"base:"}
CFGS=${CFGS:-"c5"}
for v in $VARS; do
  name=${v%%:*}; flags=${v#*:}; flags=${flags//_-D/ -D}
  [ "$name" = base ] || python -m paper_1402_4381_b200.build --out paper_1402_4381_b200/tune_$name.so $flags > /dev/null
done
lib() { [ "$1" = base ] && echo paper_1402_4381_b200/libct_oslalm.so || echo paper_1402_4381_b200/tune_$1.so; }
for c in $CFGS; do for v in $VARS; do name=${v%%:*}
  CT_OSLALM_LIB=$(lib $name) python tools/time_iter.py $c 1
done; done
