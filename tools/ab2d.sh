# A/B timing of 2D tuning variants (same box, same call): projector pair and the c2 bench step
python -c "import __graft_entry__ as g; g.build()"
VARS=${VARS:-"base: F5:-DCT_FWD2D_MINB=5 B5:-DCT_BACK2D_MINB=5"}
for v in $VARS; do
  name=${v%%:*}; flags=${v#*:}
  [ "$name" = base ] || python -m paper_1402_4381_b200.build --out paper_1402_4381_b200/tune_$name.so $flags > /dev/null
done
lib() { [ "$1" = base ] && echo paper_1402_4381_b200/libct_oslalm.so || echo paper_1402_4381_b200/tune_$1.so; }
for r in 1 2; do for v in $VARS; do name=${v%%:*}
  CT_OSLALM_LIB=$(lib $name) python tools/time_proj.py c2 30
  CT_OSLALM_LIB=$(lib $name) python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_ms']; print('$name', 'bench', f\"{d['value']:.4g}\", {s: round(v['ms_total']/v['launches']*1e3, 1) for s, v in k.items()})"
done; done
