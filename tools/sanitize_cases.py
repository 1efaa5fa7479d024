"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): every
kernel family of the library through the C ABI on tiny inputs.
python tools/sanitize_cases.py   (run as: compute-sanitizer --tool racecheck python tools/sanitize_cases.py)"""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1402_4381_b200 import ctlib  # noqa: E402
from paper_1402_4381_b200 import inputs as I  # noqa: E402
from tests import geomutil as GU  # noqa: E402

torch.manual_seed(0)


def oslalm(g, nbr, M=4, iters=2, cfg=None, inner="sqs", n_inner=1, bb=False):
    geo = ctlib.Geometry(g)
    if cfg is not None:
        d = I.synthesize(cfg)
        m0 = I.support_mask(cfg)
    else:
        ell = [(0.0, 0.0, 0.0, 4.0, 3.5, 2.5, 0.0, 0.02), (1.0, -0.5, 0.3, 1.2, 0.8, 0.9, 0.4, 0.01)]
        d = I.noisy_data(g, ell, 1e5, 0.0, 5)
        m0 = torch.ones(geo.img_shape, dtype=torch.uint8)
    dl, S = geo.sqs_denom(d["w"].cuda(), m0.cuda())
    sol = ctlib.OSLALM(geo, M, beta=2.0 ** 10, delta=2e-4, nbr=nbr, inner=inner, n_inner=n_inner, bb=bb)
    sol.set_data(d["y"].cuda(), d["w"].cuda(), dl, S)
    x = torch.zeros(geo.img_shape, device="cuda")
    sol.run(x, iters)
    geo.reg_grad(x, S, 2.0 ** 10, 2e-4, nbr)
    geo.count_vv(S)
    torch.cuda.synchronize()
    return geo, d


# 2D fan: fwd2d tile + finalize, back2d epilogues, K3 2D, the PDL graph; FISTA; BB; FBP
c1 = I.scaled(I.config("c1"), "c1", nx=32, ny=32, na=48)
geo, d = oslalm(c1.geom, 8, cfg=c1)
geo.fbp(d["y"].cuda())
oslalm(c1.geom, 8, cfg=c1, inner="fista", n_inner=2)
oslalm(c1.geom, 8, cfg=c1, bb=True, iters=3)
# 3D: pair-row forward H = 1 (32 < nt <= 64) and H = 2 (nt <= 32), general fwd3d (nt > 64),
# back3d NTM = 64 / 32 / 0, 26-neighbour K3, FDK
g64 = GU.geom("cone_helical", nx=12, nz=16, dx=0.9766, dz=0.625, ns=40, ds=1.0239, nt=64, dt=1.0964, na=48,
              turns=2.0, pitch=0.5)
oslalm(g64, 26)
oslalm(GU.small_geoms()["helical_c4"], 26)
g80 = GU.geom("cone_axial", nx=10, nz=12, dx=0.9766, dz=0.625, ns=30, ds=1.0239, nt=80, dt=0.4, na=24)
geo, d = oslalm(g80, 26)
geo.fbp(d["y"].cuda())
oslalm(GU.small_geoms()["axial_c3"], 26, inner="fista", n_inner=3)
# virtual ranks (row slabs and z-slabs): the exchange kernels and event ordering
for zs in (False, True):
    g = GU.small_geoms()["helical_c4"]
    from paper_1402_4381_b200 import host
    geoms = [I.slab_geom(g, *host.rank_zslab(g["nz"], r, 2)) for r in range(2)] if zs else [g, g]
    geos = [ctlib.Geometry(gg) for gg in geoms]
    ctlib.Geometry.comm_init_virtual(geos, zslab=zs)
    ell = [(0.0, 0.0, 0.0, 4.0, 3.5, 2.5, 0.0, 0.02)]
    d = I.noisy_data(g, ell, 1e5, 0.0, 5)
    yc, wc = d["y"].cuda(), d["w"].cuda()
    S = [torch.ones(gg.img_shape, dtype=torch.uint8, device="cuda") for gg in geos]
    dls = [torch.empty(gg.img_shape, device="cuda") for gg in geos]
    scr = [torch.empty(ctlib.ct_sqs_denom_scratch_bytes(gg.h), dtype=torch.uint8, device="cuda") for gg in geos]
    sols = [ctlib.OSLALM(gg, 4, beta=2.0 ** 10, delta=2e-4, nbr=26) for gg in geos]
    xs = [torch.zeros(gg.img_shape, device="cuda") for gg in geos]
    sts = [torch.cuda.Stream() for _ in geos]
    torch.cuda.synchronize()

    def work(r):
        ctlib.ct_sqs_denom(geos[r].h, wc, S[r], dls[r], scr[r], stream=sts[r])
        sols[r].set_data(yc, wc, dls[r], S[r])
        sols[r].run(xs[r], 2, stream=sts[r])

    th = [threading.Thread(target=work, args=(r,)) for r in range(2)]
    [t.start() for t in th]
    [t.join() for t in th]
    torch.cuda.synchronize()
print("sanitize cases done")
