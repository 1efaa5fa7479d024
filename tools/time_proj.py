"""Time the projector kernels of a config (one subset, CUDA events): python tools/time_proj.py c3 [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1402_4381_b200 import ctlib  # noqa: E402
from paper_1402_4381_b200 import inputs as I  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg = I.config(name)
g = cfg.geom
geo = ctlib.Geometry(g)
m = I.support_mask(cfg, device="cuda")
x = torch.rand(geo.img_shape, device="cuda") * 0.02 * m
M = cfg.M
views = (7 % M, M, (g["na"] - 7 % M + M - 1) // M)
y = torch.empty(geo.sino_shape(views[2]), device="cuda")
b = torch.empty(geo.img_shape, device="cuda")
for _ in range(2):
    ctlib.ct_fwd_proj(geo.h, views, x, y)
    ctlib.ct_back_proj(geo.h, views, y, b)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
ev[0].record()
for _ in range(reps):
    ctlib.ct_fwd_proj(geo.h, views, x, y)
ev[1].record()
for _ in range(reps):
    ctlib.ct_back_proj(geo.h, views, y, b)
ev[2].record()
torch.cuda.synchronize()
print(f"{os.environ.get('CT_OSLALM_LIB', 'default')} {name}: fwd {ev[0].elapsed_time(ev[1]) / reps:.3f} ms  "
      f"back {ev[1].elapsed_time(ev[2]) / reps:.3f} ms  checksum {float(y.sum()):.6e} {float(b.sum()):.6e}")
