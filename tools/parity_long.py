"""Long GPU-vs-oracle OS-LALM comparisons at full size (builder-run evidence, too slow for the
-m gpu suite): python tools/parity_long.py c3 20 [out.json] [nz_keep]
nz_keep: keep only the central nz_keep slices of the volume (full planes, detector and views;
the helical configs' oracle cost at full size is hours).
Writes the RMS / max difference over S (HU), the restart decisions and the rho trajectory
agreement after every iteration."""
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
from paper_1402_4381_b200 import ctlib  # noqa: E402
from paper_1402_4381_b200 import inputs as I  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
n_iter = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = sys.argv[3] if len(sys.argv) > 3 else f"gpurun_out/parity_long_{name}.json"
nz_keep = int(sys.argv[4]) if len(sys.argv) > 4 else 0
cfg = I.config(name)
if nz_keep:
    z0 = (cfg.geom["nz"] - nz_keep) // 2
    cfg = I.ScanConfig(cfg.name, I.slab_geom(cfg.geom, z0, z0 + nz_keep), cfg.M, cfg.n_iter, cfg.beta, cfg.delta,
                       cfg.nbr, cfg.I0, cfg.sigma, cfg.recipe, cfg.body_z, dict(cfg.extra))
g = cfg.geom
d = I.synthesize(cfg, device="cuda", views_per_chunk=8 if not cfg.is2d else 128)
m0 = I.support_mask(cfg, device="cuda")
geo = ctlib.Geometry(g)
dl, S = geo.sqs_denom(d["w"], m0)
sol = ctlib.OSLALM(geo, cfg.M, beta=cfg.beta, delta=cfg.delta, nbr=cfg.nbr)
sol.set_data(d["y"], d["w"], dl, S)
x = torch.zeros(geo.img_shape, device="cuda")
xs, logs = [], []
for it in range(n_iter):
    logs += sol.run(x, 1, log=True)
    xs.append(I.to_oracle_image(x.cpu().numpy()).astype(np.float32))
yo, wo = I.to_oracle_sino(d["y"].cpu()), I.to_oracle_sino(d["w"].cpu())
del d, sol, dl, x
torch.cuda.empty_cache()
t0 = time.time()
dlo, So = O.sqs_denom(g, wo, I.to_oracle_image(m0.cpu()).astype(np.uint8))
assert np.array_equal(I.to_oracle_image(S.cpu().numpy()).astype(np.uint8), So)
xo, logo, _, _ = O.oslalm_run(g, yo, wo, dlo, So, np.zeros(O.img_shape(g)), M=cfg.M, beta=cfg.beta,
                              delta=cfg.delta, nbr=cfg.nbr, n_iter=n_iter)
t_or = time.time() - t0
log = np.array(logs)
Sm = So > 0
xg = xs[-1]
res = {"config": name, "nz_keep": nz_keep or cfg.geom.get("nz", 1), "iters": n_iter, "M": cfg.M,
       "rms_HU": math.sqrt(((xg - xo)[Sm] ** 2).mean()) / I.HU,
       "max_abs_HU": float(np.abs(xg - xo)[Sm].max() / I.HU),
       "image_rms_HU": math.sqrt((xo[Sm] ** 2).mean()) / I.HU,
       "restarts_gpu": int(log[:, 2].sum()), "restarts_oracle": int(logo[:, 2].sum()),
       "restart_decisions_identical": bool(np.array_equal(log[:, 2], logo[:, 2])),
       "rho_max_rel_diff": float(np.max(np.abs(log[:, 0] - logo[:, 0]) / np.abs(logo[:, 0]))),
       "xi_sign_agreement": float(np.mean(np.sign(log[:, 1]) == np.sign(logo[:, 1]))),
       "oracle_seconds": t_or, "host_cores": os.cpu_count(),
       "gpu_change_per_iter_HU": [math.sqrt(((xs[i] - xs[i - 1])[Sm] ** 2).mean()) / I.HU for i in range(1, n_iter)]}
os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
with open(out, "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps({k: v for k, v in res.items() if k != "gpu_change_per_iter_HU"}))
