"""Per-launch DRAM traffic of the bench's kernel steps from one `ncu --set full` capture.

usage: python tools/ncu_traffic.py rep.ncu-rep CONFIG_ID OUT.json
Writes {CONFIG_ID: {step: {"bytes_per_launch": B, "kernels": {...}, "src": rep}}} merged into OUT.json.
A bench step may be several kernels (fwd_resid = fwd2d_tile + fwd2d_finalize): their averages add.
bench.py reports `roofline.traffic` from this file (profiles/traffic.json) for its dominant step.
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

STEPS = {   # bench step -> kernel-name prefixes
    "fwd_resid": ("fwd2d_tile_kernel", "fwd2d_finalize_kernel", "fwd3d_kernel", "fwd3d2_kernel"),
    "back_gupd": ("back2d_kernel", "back3d_kernel"),
    "sqs_update": ("sqs_update_kernel", "sqs_update2d_kernel", "sqs_update3d_kernel"),
}


def main():
    rep, cfg, out = sys.argv[1], sys.argv[2], sys.argv[3]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    kn, rd, wr = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
    units = rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    per = defaultdict(list)
    for r in rows[2:]:
        name = r[kn].split("(")[0].split("<")[0].replace("void ", "").replace("ct::", "").strip()
        b = float(r[rd]) * scale[units[rd]] + float(r[wr]) * scale[units[wr]]
        per[name].append(b)
    res = {}
    for step, prefixes in STEPS.items():
        ks = {k: sum(v) / len(v) for k, v in per.items() if k.startswith(prefixes)}
        if ks:
            res[step] = {"bytes_per_launch": sum(ks.values()), "kernels": ks, "src": os.path.basename(rep)}
    data = {}
    if os.path.exists(out):
        with open(out) as f:
            data = json.load(f)
    data[cfg] = res
    with open(out, "w") as f:
        json.dump(data, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
