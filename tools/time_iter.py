"""Per-kernel times of OS-LALM iterations as the bench runs them (state path: column trimming,
fused residual / g-update epilogues), CUDA events around every kernel on the launching stream:
python tools/time_iter.py c5 [iters]   (CT_OSLALM_LIB selects a tuning variant)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1402_4381_b200 import ctlib  # noqa: E402
from paper_1402_4381_b200 import inputs as I  # noqa: E402

if os.environ.get("CT_L2_PERSIST_MB"):   # experiment: L2 set-aside for evict_last / persisting accesses
    import ctypes
    import glob
    torch.zeros(1, device="cuda")
    rt = ctypes.CDLL(sorted(glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*")) +
                            glob.glob("/usr/local/cuda/lib64/libcudart.so*"))[0])
    rc = rt.cudaDeviceSetLimit(6, ctypes.c_size_t(int(os.environ["CT_L2_PERSIST_MB"]) << 20))   # cudaLimitPersistingL2CacheSize
    print("persisting L2 limit rc", rc, file=sys.stderr)
name = sys.argv[1] if len(sys.argv) > 1 else "c5"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = I.config(name)
d = I.synthesize(cfg, device="cuda", views_per_chunk=8 if not cfg.is2d else 128)
geo = ctlib.Geometry(cfg.geom)
dl, S = geo.sqs_denom(d["w"], I.support_mask(cfg, device="cuda"))
sol = ctlib.OSLALM(geo, cfg.M, beta=cfg.beta, delta=cfg.delta, nbr=cfg.nbr)
sol.set_data(d["y"], d["w"], dl, S)
x = torch.zeros(geo.img_shape, device="cuda")
sol.iterate(x)
sol.iterate(x)
sol.set_timing(True)
for _ in range(iters):
    sol.iterate(x)
torch.cuda.synchronize()
t = sol.timing()
print(f"{os.path.basename(os.environ.get('CT_OSLALM_LIB', 'default'))} {name}: " +
      "  ".join(f"{k} {v[0] / max(v[1], 1):.3f} ms" for k, v in t.items() if v[1]) + f"  sum(x) {float(x.sum()):.6e}")
