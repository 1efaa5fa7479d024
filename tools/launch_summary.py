"""Per-kernel aggregate of an ncu launch list (`--metrics gpu__time_duration.sum --csv`).
usage: python tools/launch_summary.py launches.csv [header line]"""
import csv
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    kn, mn, mv, un = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
    per = defaultdict(list)
    for r in rows[1:]:
        if r[mn] != "gpu__time_duration.sum":
            continue
        per[r[kn].split("(")[0]].append(float(r[mv].replace(",", "")) * scale[r[un]])
    tot = sum(sum(v) for v in per.values())
    if len(sys.argv) > 2:
        print(sys.argv[2])
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k[:60]:60s} n={len(v):5d} avg={sum(v) / len(v):9.2f}us share={100 * sum(v) / tot:5.1f}%")


if __name__ == "__main__":
    main()
