# A/B of build variants on the bench's own step kernels (same box, same call):
#   VARS="name:-DFLAG=V[_-DFLAG2=V2] ..." (base = default build)  CFGS="c2 c5"  ITERS=2
python -c "import __graft_entry__ as g; g.build()"
VARS=${VARS:-"base:"}
CFGS=${CFGS:-"c2"}
for v in $VARS; do
  name=${v%%:*}; flags=${v#*:}; flags=${flags//_-D/ -D}
  [ "$name" = base ] || python -m paper_1402_4381_b200.build --out paper_1402_4381_b200/tune_$name.so $flags > /dev/null
done
lib() { [ "$1" = base ] && echo paper_1402_4381_b200/libct_oslalm.so || echo paper_1402_4381_b200/tune_$1.so; }
for r in 1 2; do for c in $CFGS; do for v in $VARS; do name=${v%%:*}
  it=""; [ "$c" = c2 ] || it="--iters ${ITERS:-2}"
  CT_OSLALM_LIB=$(lib $name) python bench.py --config $c $it --steps 2 --warmup 3 --no-e2e --no-cpu-baseline | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_ms']; print('$c', '$name', f\"{d['value']:.4g}\", {s: round(v['ms_total']/v['launches'], 4) for s, v in k.items()})"
done; done; done
