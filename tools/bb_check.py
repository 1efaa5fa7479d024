"""Convergence of OS-LALM with / without Barzilai-Borwein scaling (reading B-BB) on c2:
RMS difference (HU, over S) to a long plain OS-LALM run, and the fraction of S at zero."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1402_4381_b200 import ctlib, inputs as I  # noqa: E402

cfg = I.config("c2")
g = cfg.geom
d = I.synthesize(cfg)
geo = ctlib.Geometry(g)
dl, S = geo.sqs_denom(d["w"].cuda(), I.support_mask(cfg).cuda())
on = S > 0


def run(n, **kw):
    sol = ctlib.OSLALM(geo, cfg.M, beta=cfg.beta, delta=cfg.delta, nbr=cfg.nbr, **kw)
    sol.set_data(d["y"].cuda(), d["w"].cuda(), dl, S)
    x = torch.zeros(geo.img_shape, device="cuda")
    snaps = {}
    for it in range(1, n + 1):
        sol.iterate(x)
        snaps[it] = x.clone()
    return snaps, (sol.alpha() if kw.get("bb") else None)


ref, _ = run(300)
xr = ref[300]
for kw in ({}, dict(bb=True), dict(mode="fixed", rho_fixed=1.0), dict(bb=True, mode="fixed", rho_fixed=1.0),
           dict(bb=True, alpha_min=0.3)):
    snaps, a = run(30, **kw)
    row = []
    for k in (5, 10, 20, 30):
        e = float(((snaps[k] - xr)[on] ** 2).mean().sqrt()) / I.HU
        z = float((snaps[k][on] == 0).float().mean())
        row.append(f"it{k}: {e:7.2f} HU (zero {z:.2f})")
    print(kw or "plain", " | ".join(row), "alpha", a)
