"""Profiling driver: the projector kernels of one config on one subset, through the C ABI.

python tools/prof_proj.py c3 [reps]   -> fwd + back of subset 7 (41 views for c3), reps times,
then one full OS-LALM iteration (fused kernels).  Used under ncu (profiles/README.md)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1402_4381_b200 import ctlib  # noqa: E402
from paper_1402_4381_b200 import inputs as I  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = I.config(name)
g = cfg.geom
geo = ctlib.Geometry(g)
m = I.support_mask(cfg, device="cuda")
x = torch.rand(geo.img_shape, device="cuda") * 0.02 * m
views = (7 % cfg.M, cfg.M, (g["na"] - 7 % cfg.M + cfg.M - 1) // cfg.M)
y = torch.empty(geo.sino_shape(views[2]), device="cuda")
b = torch.empty(geo.img_shape, device="cuda")
for _ in range(reps):
    ctlib.ct_fwd_proj(geo.h, views, x, y)
    ctlib.ct_back_proj(geo.h, views, y, b)
torch.cuda.synchronize()
print("ok", name, float(y.abs().sum()), float(b.abs().sum()))
