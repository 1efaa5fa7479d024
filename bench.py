#!/usr/bin/env python
"""bench.py — OS-LALM CT hot path on B200 (BASELINE.json metric).

A step = one OS-LALM outer iteration (BASELINE.md T_iter) of the chosen config (default c5 =
BASELINE configs[4], the helical scaling config the metric is quoted on at 1/2/4/8 GPUs):
M inner steps, each K3 update, K1 forward projection + fused weighted residual, K2
back-projection + fused g-update / xi, K4 rho continuation.  The setup (D_L = A'WA1, the
support, the initial image) runs once before the warm-up and is reported as setup_ms.
The W warm-up and K timed steps are iterations 1..W and W+1..W+K of one reconstruction.
Inputs are synthetic (seeded phantom, Poisson noise) and resident in HBM.

value  = voxel-ray updates/s = 2 U (one forward and one back-projection of every view per
         iteration, U = #(view, voxel in S) pairs with a non-empty footprint) / T_iter.
iters_per_s = 1 / T_iter.

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]
--gpus N > 1 launches itself under torch.distributed.run when WORLD_SIZE is unset (one rank
per GPU); views of every subset are split into contiguous blocks per rank and the partial
back-projections are reduce-scattered with NCCL (strong scaling); --zslab selects the
z-slab decomposition instead.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

METRIC = "voxel-ray updates/s (fwd+back proj)"
UNIT = "voxel-ray updates/s"
FP32_LANES_PER_SM = 128
N_SM = 148


def peaks():
    p = {"hbm_gbs": 6553.0, "sm_max_mhz": 1965.0, "src": "fallback"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        p.update(hbm_gbs=float(mp["hbm_gbs"]), sm_max_mhz=float(mp.get("sm_max_mhz", 1965.0)), src="measured")
    except Exception:
        pass
    # FP32 ALU peak derived from unit counts and the max SM clock
    p["fp32_tflops"] = N_SM * FP32_LANES_PER_SM * 2 * p["sm_max_mhz"] * 1e6 / 1e12
    return p


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return ws, rank, local


def allreduce_max(v, ws):
    if ws == 1:
        return v
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def load_traffic(config_id):
    """DRAM bytes per launch of each bench step from one committed `ncu --set full` capture
    (profiles/traffic.json, written by tools/ncu_traffic.py); {} if absent."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(config_id, {})
    except Exception:
        return {}


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()


def workload_name(cfg, n_iter=None):
    g = cfg.geom
    shape = f"{g['nx']}x{g['ny']}" + ("" if cfg.is2d else f"x{g['nz']}")
    det = f"{g['ns']}ch" + ("" if cfg.is2d else f"x{g['nt']}rows")
    return (f"{cfg.name}: {g['kind']} {shape} image, {det}, {g['na']} views, M={cfg.M}; "
            f"one step = one OS-LALM outer iteration (M subset fwd/back pairs + M updates), "
            f"the config's reconstruction is {n_iter or cfg.n_iter} iterations")


# views per reference-arm step: a bounded block of one subset (whole subsets for the small configs)
REF_VIEWS = {"c1": 30, "c2": 41, "c3": 16, "c4": 24, "c5": 16}


def oracle_chunk(cfg, x, mo, i, nv):
    """One bounded oracle sample: forward + back projection of the first nv views of subset
    pi[i mod M] (fp64, OpenMP over the host cores).  Returns the voxel-ray updates done."""
    import oracle as O
    g = cfg.geom
    sub = O.bit_reversal(cfg.M)[i % cfg.M]
    cnt = min(nv, O.nviews(g, sub, cfg.M))
    p = O.fwd(g, x, sub, cfg.M, cnt)
    O.back(g, p, sub, cfg.M, cnt)
    return 2 * O.count_vv(g, mo, sub, cfg.M, cnt), cnt


def oracle_inputs(cfg):
    import oracle as O
    from paper_1402_4381_b200 import inputs as I
    O.build()
    m = I.support_mask(cfg)
    mo = I.to_oracle_image(m).astype(np.uint8)
    x = np.random.default_rng(0).random(O.img_shape(cfg.geom)) * 0.02 * mo
    return x, mo


def cpu_oracle_sample(cfg, budget_s=15.0):
    """The fp64 oracle as it stands, timed on bounded samples of the same workload."""
    x, mo = oracle_inputs(cfg)
    nv = REF_VIEWS.get(cfg.name, 32)
    done, work, views, t0 = 0, 0, 0, time.perf_counter()
    while True:
        w, c = oracle_chunk(cfg, x, mo, done, nv)
        work += w; views += c; done += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    el = time.perf_counter() - t0
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return {"value": work / el, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{done} block(s) of <= {nv} views of one subset each ({views} views) of {cfg.name}: "
                      f"forward + back projection, fp64, OpenMP; {el:.1f} s"}


def run_reference(args):
    """--impl reference: the oracle is this tier's reference arm (CPU, rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_1402_4381_b200 import inputs as I
    cfg = I.config(args.config)
    x, mo = oracle_inputs(cfg)
    nv = REF_VIEWS.get(cfg.name, 32)
    for i in range(args.warmup):
        oracle_chunk(cfg, x, mo, i, nv)
    times, work = [], 0
    for i in range(args.steps):
        t0 = time.perf_counter()
        w, _ = oracle_chunk(cfg, x, mo, args.warmup + i, nv)
        times.append(time.perf_counter() - t0)
        work += w
    T = sum(times)
    value = work / T
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    sample = f"per step: forward + back projection of the first <= {nv} views of one subset of {cfg.name} (fp64)"
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": workload_name(cfg) + f" [reference step: {nv} views of one subset, fwd+back]",
                      "config_id": cfg.name},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    return 0


def spawn_ranks(n):
    """--gpus N without a torchrun environment: re-launch this command under
    torch.distributed.run with one rank per GPU (rendezvous on 127.0.0.1)."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20, help="timed OS-LALM outer iterations")
    ap.add_argument("--warmup", type=int, default=3, help="untimed iterations before the timed ones")
    ap.add_argument("--config", default="c5")
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--inner", default="sqs", choices=("sqs", "fista"), help="inner solver (NEXT-1: fista)")
    ap.add_argument("--n-inner", type=int, default=1, help="inner FISTA iterations (with --inner fista)")
    ap.add_argument("--bb", action="store_true", help="Barzilai-Borwein scaling of the SQS Hessian (NEXT-2)")
    ap.add_argument("--zslab", action="store_true",
                    help="cone beam: z-slab decomposition over the ranks, partial sinograms summed (NEXT-3)")
    ap.add_argument("--init", default="zero", choices=("zero", "fbp"),
                    help="initial image: zero on S (G10) or the FBP/FDK image (NEXT-4, P:586)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)

    ws, rank, local = dist_setup()
    torch.cuda.set_device(local)
    from paper_1402_4381_b200 import build, ctlib
    from paper_1402_4381_b200 import inputs as I
    if rank == 0:
        build.build()
    if ws > 1:
        barrier(ws)
    ctlib.load()
    cfg = I.config(args.config)
    g = cfg.geom
    dev = torch.device("cuda", local)
    st = torch.cuda.current_stream()

    # ---- inputs (synthetic, seeded), resident in HBM
    data = I.synthesize(cfg, device=dev, views_per_chunk=8 if not cfg.is2d else 128)
    y, w = data["y"].contiguous(), data["w"].contiguous()
    del data
    m0 = I.support_mask(cfg, device=dev)
    if args.zslab:   # NEXT-3: this rank's z-slab of the volume (its own geometry)
        from paper_1402_4381_b200.host import rank_zslab
        z0, z1 = rank_zslab(g["nz"], rank, ws)
        g = I.slab_geom(g, z0, z1)
        m0 = m0[..., z0:z1].contiguous()
    geo = ctlib.Geometry(g, local)
    if ws > 1 or args.zslab:
        import torch.distributed as dist
        uid = [ctlib.ct_comm_get_unique_id() if rank == 0 else None]
        if ws > 1:
            dist.broadcast_object_list(uid, src=0)
        geo.comm_init(rank, ws, uid[0], zslab=args.zslab)
    mask = m0.clone()
    dl = torch.empty(geo.img_shape, dtype=torch.float32, device=dev)
    scratch = torch.empty(ctlib.ct_sqs_denom_scratch_bytes(geo.h), dtype=torch.uint8, device=dev)
    x = torch.zeros(geo.img_shape, dtype=torch.float32, device=dev)
    sol = ctlib.OSLALM(geo, cfg.M, beta=cfg.beta, delta=cfg.delta, nbr=cfg.nbr, inner=args.inner,
                       n_inner=args.n_inner, bb=args.bb)
    sol.set_data(y, w, dl, mask)
    N = int(np.prod(geo.img_shape))
    ws_bytes = (y.numel() + w.numel() + 6 * N) * 4        # y, W and the image-sized state
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev) if ws_bytes < 4 * l2_bytes else None

    # ---- setup (reported separately): D_L = A'WA1 and the support (S8), the initial image
    def setup():
        mask.copy_(m0)
        ctlib.ct_sqs_denom(geo.h, w, mask, dl, scratch)
        sol.reset()
        if args.init == "fbp":
            fs = torch.empty(ctlib.ct_fbp_scratch_bytes(geo.h), dtype=torch.uint8, device=dev)
            ctlib.ct_fbp(geo.h, y, x, fs)
        else:
            x.zero_()

    setup()                                      # untimed first call (lazy module / smem setup)
    barrier(ws)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    setup()
    e1.record(st)
    barrier(ws)
    setup_ms = allreduce_max(e0.elapsed_time(e1), ws)

    # ---- work counts (fp64 geometry on the device; outside any timed region)
    U, nnz, C = geo.counts(mask)
    work_step = 2 * U                            # one forward + one back-projection of every view
    local_counts = (nnz, U, C)                   # this rank's geometry (a slab's voxels with --zslab)
    if args.zslab and ws > 1:                    # the slabs partition the voxels: the job's work is their sum
        import torch.distributed as dist
        t = torch.tensor([work_step, U, nnz], dtype=torch.float64, device=dev)
        dist.all_reduce(t)
        work_step, U, nnz = (int(v) for v in t.tolist())

    # ---- warm-up iterations (the first computes the initial subset gradient and captures the
    # CUDA graph); the clock sampler starts here so that it samples the timed region
    clk = ClockSampler(local).__enter__()
    for _ in range(max(args.warmup, 1)):
        sol.iterate(x)
    barrier(ws)

    # ---- timed region: K outer iterations (iterations W+1 .. W+K of one reconstruction)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    l0 = ctlib.ct_kernel_launches()
    try:
        barrier(ws)
        for i in range(args.steps):
            if flush is not None:
                flush.zero_()
            starts[i].record(st)
            sol.iterate(x)
            ends[i].record(st)
        barrier(ws)
    finally:
        clk.__exit__(None, None, None)
    launches = ctlib.ct_kernel_launches() - l0
    T = sum(s.elapsed_time(e) for s, e in zip(starts, ends)) / 1e3
    T = allreduce_max(T, ws)
    value = work_step * args.steps / T

    # forward-projection trimming skips voxel columns whose x is zero along a whole image line
    # end: the S voxels in all-zero columns bound the work counted but not executed
    colzero = (x == 0).all(dim=2) & (mask != 0).any(dim=2)
    skipped_frac = float((mask.sum(dim=2) * colzero).sum().item()) / max(1.0, float(mask.sum().item()))

    # ---- per-kernel timing pass: one more iteration with CUDA events around every kernel on
    # the launching stream (eager launches, no graph)
    sol.set_timing(True)
    if flush is not None:
        flush.zero_()
    sol.iterate(x)
    torch.cuda.synchronize()
    kt = sol.timing()
    sol.set_timing(False)
    pk = peaks()
    M = cfg.M
    # algorithmic FLOPs per projection launch: 2 nnz + 15 U + 150 C, per subset = full / M
    lnnz, lU, lC = local_counts
    share = 1 if args.zslab else ws
    flop_launch = (2 * lnnz + 15 * lU + 150 * lC) / M / share
    dom = max(("fwd_resid", "back_gupd"), key=lambda k: kt[k][0])
    ms_launch = kt[dom][0] / max(kt[dom][1], 1)
    achieved = flop_launch / (ms_launch / 1e3) / 1e12
    total_kt = sum(v[0] for v in kt.values())
    upd_ms = kt["sqs_update"][0] / max(kt["sqs_update"][1], 1)
    # x, G, g, D_L read (16 B) + mask (1 B) + x' write (4 B) per updated voxel (row-slab ranks update N/P)
    upd_bytes = 21 * N / (ws if (ws > 1 and not args.zslab and args.inner == "sqs") else 1)
    traffic = load_traffic(cfg.name)
    roofline_alu = {"bound": "alu", "kernel": dom, "achieved": achieved, "peak": pk["fp32_tflops"], "unit": "TFLOP/s",
                "frac": achieved / pk["fp32_tflops"], "traffic": traffic.get(dom, {}).get("bytes_per_launch"),
                "traffic_src": traffic.get(dom, {}).get("src"),
                "peak_src": f"derived: {N_SM} SM x {FP32_LANES_PER_SM} FP32 lanes x 2 x {pk['sm_max_mhz']:.0f} MHz",
                "flop_per_launch": flop_launch, "ms_per_launch": ms_launch,
                "share_of_step": kt[dom][0] / total_kt}
    # the projector's compulsory DRAM bytes per launch: the image once + the subset sinogram
    # (y, W read, residual written and read back by the back-projector)
    cells_sub = (g["na"] // M) * g["ns"] * (1 if cfg.is2d else g["nt"])
    roofline_alu["algorithmic_dram_bytes"] = 4 * N + 16 * cells_sub
    streaming = {"bound": "hbm", "kernel": "sqs_update", "achieved": upd_bytes / (upd_ms / 1e3) / 1e9,
                 "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": upd_bytes / (upd_ms / 1e3) / 1e9 / pk["hbm_gbs"],
                 "traffic": traffic.get("sqs_update", {}).get("bytes_per_launch"), "bytes_per_launch": upd_bytes,
                 "ms_per_launch": upd_ms}
    kernel_ms = {k: {"ms_total": v[0], "launches": v[1], "share": v[0] / total_kt} for k, v in kt.items() if v[1]}
    # BASELINE.json's "HBM/L2 gather roofline": every nonzero's operand fetched
    # through L2 once, T = max(T_HBM, 4 B nnz / BW_L2), BW_L2 = L2-resident read bandwidth
    # measured here (no vendor number available)
    l2 = ctlib.ct_peak_l2_read(local)
    gather_bytes = 4.0 * lnnz / M / share
    rg = {}
    for k in ("fwd_resid", "back_gupd"):
        ms_k = kt[k][0] / max(kt[k][1], 1)
        rg[k] = {"achieved": gather_bytes / (ms_k / 1e3) / 1e9, "frac": gather_bytes / (ms_k / 1e3) / 1e9 / l2,
                 "ms_per_launch": ms_k}
    # the projector pair (BASELINE.json's "projector pair reaching >= 50 % of the HBM/L2 gather
    # roofline"): both launches move the same gather bytes, so the pair's fraction is
    # 2 B / (t_fwd + t_back) / BW_L2
    ms_pair = rg["fwd_resid"]["ms_per_launch"] + rg["back_gupd"]["ms_per_launch"]
    pair_frac = 2 * gather_bytes / (ms_pair / 1e3) / 1e9 / l2
    # primary roofline: the BASELINE-named L2 gather roofline of the dominant kernel (SURVEY
    # §8(d): "BJ's >= 50 % target on 1 B200 is judged against this"); the ALU roofline and
    # SURVEY's tighter bound max(T_alu, T_gather(smem), T_HBM) beside it
    roofline = {"bound": "l2-gather", "kernel": dom, "achieved": rg[dom]["achieved"],
                "peak": l2, "unit": "GB/s", "frac": rg[dom]["frac"], "pair_frac": pair_frac, "per_kernel": rg,
                "bytes_per_launch": gather_bytes, "ms_per_launch": rg[dom]["ms_per_launch"],
                "traffic": roofline_alu["traffic"], "traffic_src": roofline_alu["traffic_src"],
                "algorithmic_dram_bytes": roofline_alu["algorithmic_dram_bytes"],
                "share_of_step": roofline_alu["share_of_step"],
                "peak_src": "measured in this run: ct_peak_l2_read (48 MiB buffer streamed 200x, float4 loads)",
                "note": "4 B per nonzero through L2 once (SURVEY 8(d)); traffic = ncu DRAM bytes of the kernel"}
    smem_tbs = N_SM * 128 * pk["sm_max_mhz"] * 1e6 / 1e12   # 128 B/clk/SM shared-memory bandwidth (derived)
    t_alu = flop_launch / (pk["fp32_tflops"] * 1e12)
    t_smem = gather_bytes / (smem_tbs * 1e12)
    t_hbm = roofline_alu["algorithmic_dram_bytes"] / (pk["hbm_gbs"] * 1e9)
    t_true = max(t_alu, t_smem, t_hbm)
    roofline_true = {"bound": ("alu" if t_true == t_alu else "smem-gather" if t_true == t_smem else "hbm"),
                     "kernel": dom, "t_bound_ms": t_true * 1e3, "ms_per_launch": ms_launch,
                     "frac": t_true * 1e3 / ms_launch, "t_alu_ms": t_alu * 1e3, "t_smem_gather_ms": t_smem * 1e3,
                     "t_hbm_ms": t_hbm * 1e3,
                     "peak_src": f"smem {smem_tbs:.1f} TB/s derived: {N_SM} SM x 128 B/clk x {pk['sm_max_mhz']:.0f} MHz"}

    # ---- end to end through the C ABI: every step copies that step's inputs (y, W) from pinned
    # host memory to the device and reads the iterate back, inside the timed region.  Without
    # an L2 flush between steps the copies are pipelined: a copy stream uploads step k + 1's
    # inputs into the other of two device buffer sets while step k computes, and reads step
    # k's iterate (a device snapshot) back while step k + 1 computes; the timed region runs
    # from the first upload to the last read-back.
    e2e = None
    if not args.no_e2e:
        y_h = y.cpu().pin_memory(); w_h = w.cpu().pin_memory()
        x_h = torch.empty(x.shape, dtype=torch.float32).pin_memory()
        bufs = [(torch.empty_like(y), torch.empty_like(w)) for _ in range(2)]
        # row-slab ranks read only their contiguous block of every subset's views: copy those
        # (view by view, each a contiguous pinned block); one rank / z-slabs copy everything
        owned = None
        if ws > 1 and not args.zslab:
            from paper_1402_4381_b200.host import rank_view_block
            owned = []
            for m in range(cfg.M):
                k0, n = rank_view_block((g["na"] - m + cfg.M - 1) // cfg.M, rank, ws)
                owned += [m + (k0 + k) * cfg.M for k in range(n)]

        def h2d(yb, wb):
            if owned is None:
                yb.copy_(y_h, non_blocking=True)
                wb.copy_(w_h, non_blocking=True)
                return y.numel() * 4 + w.numel() * 4
            for v in owned:
                yb[v].copy_(y_h[v], non_blocking=True)
                wb[v].copy_(w_h[v], non_blocking=True)
            return 2 * len(owned) * y[0].numel() * 4

        for yb, wb in bufs:                      # capture a graph per buffer set (untimed)
            h2d(yb, wb)
            sol.set_data(yb, wb, dl, mask)
            sol.iterate(x)
        x_h.copy_(x)
        torch.cuda.synchronize()
        h2d_bytes = 0
        K = args.steps
        if flush is None:
            cs = torch.cuda.Stream(device=dev)
            xsnap = [torch.empty_like(x) for _ in range(2)]
            ready = [torch.cuda.Event() for _ in range(2)]
            done = [torch.cuda.Event() for _ in range(2)]
            back = [torch.cuda.Event() for _ in range(2)]
            e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            barrier(ws)
            e_start.record(st)
            cs.wait_stream(st)
            with torch.cuda.stream(cs):
                h2d_bytes = h2d(*bufs[0])
                ready[0].record(cs)
            for k in range(K):
                b = k % 2
                if k + 1 < K:                    # upload step k + 1's inputs meanwhile
                    with torch.cuda.stream(cs):
                        if k >= 1:
                            cs.wait_event(done[1 - b])   # step k - 1 finished with that set
                        h2d(*bufs[1 - b])
                        ready[1 - b].record(cs)
                st.wait_event(ready[b])
                sol.set_data(bufs[b][0], bufs[b][1], dl, mask)
                sol.iterate(x)
                if k >= 2:
                    st.wait_event(back[b])       # step k - 2's read-back of this snapshot is done
                xsnap[b].copy_(x)
                done[b].record(st)
                with torch.cuda.stream(cs):      # read step k's iterate back meanwhile
                    cs.wait_event(done[b])
                    x_h.copy_(xsnap[b], non_blocking=True)
                    back[b].record(cs)
            st.wait_stream(cs)
            e_end.record(st)
            barrier(ws)
            Te = e_start.elapsed_time(e_end) / 1e3
            mode = "pipelined: uploads / read-backs on a copy stream overlap the previous / next step"
        else:
            es = [torch.cuda.Event(enable_timing=True) for _ in range(2 * K)]
            barrier(ws)
            for i in range(K):
                flush.zero_()
                es[2 * i].record(st)
                h2d_bytes = h2d(*bufs[0])
                sol.set_data(bufs[0][0], bufs[0][1], dl, mask)
                sol.iterate(x)
                x_h.copy_(x, non_blocking=True)
                es[2 * i + 1].record(st)
            barrier(ws)
            Te = sum(es[2 * i].elapsed_time(es[2 * i + 1]) for i in range(K)) / 1e3
            mode = "serial (L2 flushed between steps)"
        Te = allreduce_max(Te, ws)
        torch.cuda.synchronize()
        e2e = {"value": work_step * K / Te, "unit": UNIT,
               "h2d_bytes_per_step": int(h2d_bytes), "d2h_bytes_per_step": int(x.numel() * 4),
               "ms_per_step": 1e3 * Te / K, "copies": mode,
               # the last read-back is the final iterate (the pipeline's ordering check)
               "readback_matches_device": bool(torch.equal(x_h, x.cpu()))}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_oracle_sample(cfg, args.cpu_budget)
        except Exception as e:  # the baseline is reported, never required
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle", "sample": f"failed: {e}"}

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "iters_per_s": args.steps / T, "setup_ms": setup_ms,
            "config": {"workload": workload_name(cfg), "config_id": cfg.name, "M": cfg.M, "n_iter": cfg.n_iter,
                       "step": "one OS-LALM outer iteration", "timed_iterations": f"{args.warmup + 1}..{args.warmup + args.steps}",
                       "inner": f"{args.inner} x{args.n_inner}" + (" + BB" if args.bb else ""), "init": args.init,
                       "views_per_subset": (g["na"] + cfg.M - 1) // cfg.M, "U_full_scan": U,
                       "nnz_full_scan": nnz, "work_per_step": work_step,
                       "work_skipped_frac_bound": skipped_frac,
                       "setup": "D_L = A'WA1 + support + initial image, timed separately (setup_ms)",
                       "l2": ("flushed between steps (512 MiB write, untimed)" if flush is not None else
                              f"inputs larger than L2 ({ws_bytes / 1e9:.2f} GB vs {l2_bytes / 1e6:.0f} MB); no flush"),
                       "parallelism": (f"z-slabs over {ws} GPU(s): partial sinograms all-reduced, slab "
                                       "back-projection and update, 1-slice halos" if args.zslab else
                                       f"views of each subset split over {ws} GPU(s), image row slabs; G+ and x+ "
                                       "exchanged " + ("as z-band blocks (band-limited, helical)" if g["kind"] == "cone_helical"
                                                       else "by NCCL reduce-scatter / all-gather")
                                       if ws > 1 else "1 GPU")},
            "gpu_launches": int(launches), "roofline": roofline, "roofline_alu": roofline_alu,
            "roofline_true": roofline_true, "roofline_streaming": streaming,
            "kernel_ms": kernel_ms, "clocks": clk.summary(), "e2e": e2e, "cpu_baseline": cpu,
            "peaks": {"fp32_tflops": pk["fp32_tflops"], "hbm_gbs": pk["hbm_gbs"], "src": pk["src"]},
            "build": ctlib.ct_build_info(),
        }
        print(json.dumps(out))
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
