"""OS-LALM iterations of a config through the C ABI (graph replay), for ncu captures of the
step kernels as the bench runs them:  python tools/prof_iter.py c5 [iters]
Launch order of the 3D step kernels: D_L setup fwd/back (1 each), initial subset gradient
(1 each), then per iteration M x (sqs_update, fwd, back)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1402_4381_b200 import ctlib  # noqa: E402
from paper_1402_4381_b200 import inputs as I  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = I.config(name)
d = I.synthesize(cfg, device="cuda", views_per_chunk=8 if not cfg.is2d else 128)
geo = ctlib.Geometry(cfg.geom)
dl, S = geo.sqs_denom(d["w"], I.support_mask(cfg, device="cuda"))
sol = ctlib.OSLALM(geo, cfg.M, beta=cfg.beta, delta=cfg.delta, nbr=cfg.nbr)
sol.set_data(d["y"], d["w"], dl, S)
x = torch.zeros(geo.img_shape, device="cuda")
for _ in range(iters):
    sol.iterate(x)
torch.cuda.synchronize()
print("ok", name, iters, float(x.sum()))
