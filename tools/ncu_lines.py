"""Aggregate an ncu 'source' page (--print-source cuda,sass --csv) by CUDA source line.
usage: ncu -i rep --page source --csv --print-source cuda,sass -k regex:K | python tools/ncu_lines.py [N]"""
import csv
import sys
from collections import defaultdict

N = int(sys.argv[1]) if len(sys.argv) > 1 else 25
rows = list(csv.reader(sys.stdin))
agg = defaultdict(lambda: [0.0, 0.0])
src = {}
fname = ""
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ie = hdr.index("Instructions Executed")
        ws = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) <= ie:
        continue
    try:
        line = int(r[0])
        n = float(r[ie] or 0); w = float(r[ws] or 0)
    except ValueError:
        continue
    key = (fname, line)
    agg[key][0] += n; agg[key][1] += w
    src[key] = r[1][:100]
tot_i = sum(v[0] for v in agg.values()); tot_s = sum(v[1] for v in agg.values())
print(f"total warp-instr {tot_i:.3e}  stall samples {tot_s:.0f}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:N]:
    print(f"{100*v[0]/tot_i:5.1f}% inst {100*v[1]/max(tot_s,1):5.1f}% samp  {k[0]}:{k[1]}  {src[k]}")
