"""Pins for the oracle's SQS denominator, Fair regulariser and OS-LALM loop.

PAPER.md: P:380-397 (eq. os_lalm_iterates), P:495-516 (restart indicator xi and the
rho_l schedule), P:521-537 (PWLS CT problem, substitution, L_diag = diag{A'WA1},
bit-reversal order, n-step FISTA inner solve).  Readings O4-O7, G3, G6-G14 in
DESIGN.md.  Each pin checks the oracle against an independent computation:
dense matrices built from unit vectors, finite differences, a separately written
OS-SQS loop, a separately written Python OS-LALM loop, the paper's closed-form
damping analysis, and a brute-force minimiser of a 16x16 problem.
"""
import json
import math
import os

import numpy as np
import pytest
import scipy.optimize

import oracle as O
from paper_1402_4381_b200 import inputs as I
from tests import geomutil as GU

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- paper values

def test_bit_reversal_golden():
    """Bit-reversal order with the pad-to-2^k-and-drop rule (G11)."""
    gold = json.load(open(os.path.join(GOLD, "bit_reversal.json")))
    for M, order in gold["orders"].items():
        assert O.bit_reversal(int(M)) == order
    for M in range(1, 70):
        assert sorted(O.bit_reversal(M)) == list(range(M))


def test_rho_l_schedule():
    """rho_l: rho_0 = 1, formula for l >= 1, floor rho_min = 1e-3."""
    gold = json.load(open(os.path.join(GOLD, "paper_values.json")))
    assert O.rho_l(0) == 1.0
    # l = 1: (pi/2) sqrt(1 - (pi/4)^2) ~= 0.9723
    assert abs(O.rho_l(1) - gold["rho_1_approx"]) < 5e-5
    r = [O.rho_l(l) for l in range(1, 4000)]
    assert all(a >= b for a, b in zip(r, r[1:]))                     # non-increasing
    assert min(r) == gold["rho_min"]
    first_floor = 1 + next(i for i, v in enumerate(r) if v == gold["rho_min"])
    # pi/(l+1) sqrt(1-(pi/(2l+2))^2) < 1e-3  <=>  l+1 > ~pi/1e-3
    assert first_floor == math.floor(math.pi / 1e-3 - 1) + 1 or first_floor == math.ceil(math.pi / 1e-3 - 1)
    # the ideal critical rho for a restart period r is exactly what the formula
    # gives at l = r - 1: 2 sqrt(q^2(1-q^2)) with q = pi/(2r)
    for rr in (2, 5, 17, 300):
        q = math.pi / (2 * rr)
        assert abs(O.rho_l(rr - 1) - 2 * math.sqrt(q * q * (1 - q * q))) < 1e-14


def test_max_subset_rules():
    """Max-subset rules: the GEPP axial scan (984 views, s_axial=40) gives 'about 24'."""
    from paper_1402_4381_b200 import host
    gold = json.load(open(os.path.join(GOLD, "paper_values.json")))
    assert host.max_subsets_axial(984, 40) == gold["gepp_max_subsets"]
    assert host.max_subsets_helical(984, 541.0, 949.0, 0.5, 24) == 46
    assert host.max_subsets_helical(984, 541.0, 949.0, 1.0, 24) == 23   # inversely prop. to pitch
    assert host.max_subsets_axial(40, 40) == 1


def test_damping_recurrence_reading_G6():
    """simulated per-component rate equals max|root| of the characteristic
    polynomial; critical damping closed form holds; the printed
    under-damped 'rate' is the real part, not the modulus (reading G6)."""
    def simulate(lam, rho, n=20000, tail=18000):
        """Asymptotic per-step contraction of (x, g) under P:428-434 (L = 1), renormalised."""
        x, g = 1.0, 0.3
        logs = []
        for _ in range(n):
            x = x - (lam * x + (1 / rho - 1) * g)
            g = rho / (rho + 1) * lam * x + g / (rho + 1)
            nrm = math.hypot(x, g)
            logs.append(math.log(nrm))
            x, g = x / nrm, g / nrm
        return math.exp(sum(logs[-tail:]) / tail)

    for lam, rho in ((0.25, 1.0), (0.25, 0.2), (0.1, 0.5), (0.05, 0.01), (0.5, 1.0)):
        roots = np.roots([1 + rho, -2 * (1 - lam + rho / 2), 1 - lam])
        sim = simulate(lam, rho)
        assert abs(sim - np.abs(roots).max()) < 1e-3
    lam = 0.5
    rc = 2 * math.sqrt(lam * (1 - lam))                      # rho_c = 1
    assert abs(math.sqrt((1 - lam) / (1 + rc)) - 0.5) < 1e-12  # r^c
    lam, rho = 0.25, 0.2                                      # under-damped
    printed = (1 - lam + rho / 2) / (1 + rho)
    modulus = math.sqrt((1 - lam) / (1 + rho))
    assert abs(simulate(lam, rho) - modulus) < 1e-3 and abs(printed - modulus) > 0.05


# ---------------------------------------------------------------- D_L and SQS

def _small_problem(seed=11):
    g = GU.geom("fan2d", nx=16, dx=8.0, ns=24, ds=14.0, na=36)
    ell = [(0.0, 0.0, 0.0, 55.0, 45.0, float("inf"), 0.3, 0.02),
           (15.0, -10.0, 0.0, 12.0, 18.0, float("inf"), 1.1, 0.01),
           (-20.0, 12.0, 0.0, 8.0, 8.0, float("inf"), 0.0, -0.015)]
    d = I.noisy_data(g, ell, 1e4, 0.0, seed)
    y = I.to_oracle_sino(d["y"]); w = I.to_oracle_sino(d["w"])
    xc = (np.arange(16) - 7.5) * 8.0
    r = np.sqrt(xc[:, None] ** 2 + xc[None, :] ** 2)
    mask = (r <= I.fov_radius(g) - g["dx"]).astype(np.uint8)[None]
    return g, y, w, mask


def _dense_A(g):
    n = g["nx"] * g["ny"]
    cols = []
    for j in range(n):
        e = np.zeros(n); e[j] = 1.0
        cols.append(O.fwd(g, e.reshape(1, g["ny"], g["nx"])).reshape(-1))
    return np.stack(cols, 1)


def test_sqs_denom_equals_dense():
    """D_L = diag{A'WA1} on S, computed with a dense A from unit-vector projections."""
    g, y, w, mask = _small_problem()
    A = _dense_A(g)
    one = mask.reshape(-1).astype(float)
    ref = A.T @ (w.reshape(-1) * (A @ one))
    dl, m2 = O.sqs_denom(g, w, mask)
    ref = np.where(m2.reshape(-1) > 0, ref, 0.0)
    assert np.abs(dl.reshape(-1) - ref).max() <= 1e-12 * ref.max()
    assert (m2.reshape(-1) <= mask.reshape(-1)).all()
    assert ((dl.reshape(-1) > 0) == (m2.reshape(-1) > 0)).all()


def test_sqs_inequality():
    """||A(x - xb)||_W^2 <= (x - xb)' D_L (x - xb) for x supported on S (SQS)."""
    g, y, w, mask = _small_problem()
    A = _dense_A(g)
    dl, m2 = O.sqs_denom(g, w, mask)
    S = m2.reshape(-1) > 0
    rng = np.random.default_rng(0)
    W = w.reshape(-1)
    worst = np.inf
    for _ in range(1000):
        d = rng.standard_normal(A.shape[1]) * S
        lhs = (W * (A @ d) ** 2).sum()
        rhs = (dl.reshape(-1) * d * d).sum()
        worst = min(worst, (rhs - lhs) / rhs)
    assert worst >= -1e-12


# ---------------------------------------------------------------- regulariser

def _pairs(shape, nbr):
    """Independent list of unordered neighbour pairs (j, k, w) of a [nz][ny][nx] grid."""
    nz, ny, nx = shape
    idx = np.arange(nz * ny * nx).reshape(shape)
    out = []
    offs = [(oz, oy, ox) for oz in (-1, 0, 1) for oy in (-1, 0, 1) for ox in (-1, 0, 1)
            if (oz, oy, ox) > (0, 0, 0) and (nbr == 26 or oz == 0)]
    for (oz, oy, ox) in offs:
        a = idx[max(0, -oz):nz - max(0, oz), max(0, -oy):ny - max(0, oy), max(0, -ox):nx - max(0, ox)]
        b = idx[max(0, oz):nz - max(0, -oz) or None, max(0, oy):ny - max(0, -oy) or None, max(0, ox):nx - max(0, -ox) or None]
        b = b[:a.shape[0], :a.shape[1], :a.shape[2]]
        out.append((a.reshape(-1), b.reshape(-1), np.full(a.size, 1 / math.sqrt(oz * oz + oy * oy + ox * ox))))
    return [np.concatenate(t) for t in zip(*out)]


def _fair(t, d):
    a = np.abs(t) / d
    return d * d * (a - np.log1p(a))


def _cases():
    g2 = GU.geom("fan2d", nx=12, ny=9, dx=1.0)
    g3 = GU.geom("cone_axial", nx=6, ny=5, nz=4, dx=1.0, dz=1.0, nt=4)
    return [(g2, 8), (g3, 26)]


@pytest.mark.parametrize("k", [0, 1])
def test_reg_value_matches_pair_sum(k):
    """R(x) = beta sum_{pairs in S} w psi(x_j - x_k), each unordered pair once (O5)."""
    g, nbr = _cases()[k]
    rng = np.random.default_rng(1)
    shape = O.img_shape(g)
    x = rng.random(shape) * 0.05
    mask = (rng.random(shape) > 0.2).astype(np.uint8)
    j, kk, w = _pairs(shape, nbr)
    both = (mask.reshape(-1)[j] > 0) & (mask.reshape(-1)[kk] > 0)
    ref = 3.0 * (w * _fair(x.reshape(-1)[j] - x.reshape(-1)[kk], 0.01) * both).sum()
    assert abs(O.reg_value(g, 3.0, 0.01, nbr, mask, x) - ref) <= 1e-12 * ref


@pytest.mark.parametrize("k", [0, 1])
def test_reg_grad_finite_differences(k):
    """grad R matches central finite differences of R; off S the gradient is 0."""
    g, nbr = _cases()[k]
    rng = np.random.default_rng(2)
    shape = O.img_shape(g)
    mask = (rng.random(shape) > 0.15).astype(np.uint8)
    for trial in range(5):
        x = rng.random(shape) * 0.05
        gr, cu = O.reg_grad(g, 2.0, 0.02, nbr, mask, x)
        h = 1e-6
        fd = np.zeros(x.size)
        for q in range(x.size):
            xp = x.copy().reshape(-1); xp[q] += h
            xm = x.copy().reshape(-1); xm[q] -= h
            fd[q] = (O.reg_value(g, 2.0, 0.02, nbr, mask, xp) - O.reg_value(g, 2.0, 0.02, nbr, mask, xm)) / (2 * h)
        fd = np.where(mask.reshape(-1) > 0, fd, 0.0)
        assert np.abs(gr.reshape(-1) - fd).max() <= 1e-5 * np.abs(fd).max()
    const = np.full(shape, 0.37)
    gr, _ = O.reg_grad(g, 2.0, 0.02, nbr, np.ones(shape, np.uint8), const)
    assert np.abs(gr).max() == 0.0


def test_fair_quadratic_limit():
    """Fair -> quadratic t^2/2 as delta -> inf."""
    g, nbr = _cases()[1]
    rng = np.random.default_rng(3)
    shape = O.img_shape(g)
    x = rng.random(shape)
    m = np.ones(shape, np.uint8)
    j, k, w = _pairs(shape, nbr)
    quad = (w * 0.5 * (x.reshape(-1)[j] - x.reshape(-1)[k]) ** 2).sum()
    d = 100 * np.abs(x.reshape(-1)[j] - x.reshape(-1)[k]).max()
    assert abs(O.reg_value(g, 1.0, d, nbr, m, x) / quad - 1) < 1e-2


@pytest.mark.parametrize("k", [0, 1])
def test_reg_curvature_majorizes(k):
    """Huber-curvature D_R majorises R: R(x) <= R(xb) + gradR(xb)'D + 1/2 D'diag(D_R(xb))D (G14, V9)."""
    g, nbr = _cases()[k]
    rng = np.random.default_rng(4)
    shape = O.img_shape(g)
    mask = (rng.random(shape) > 0.1).astype(np.uint8)
    worst = np.inf
    for trial in range(300):
        scale = 10 ** rng.uniform(-5, -1)
        xb = rng.random(shape) * scale
        d = rng.standard_normal(shape) * scale * (mask > 0)
        gr, cu = O.reg_grad(g, 1.0, 2e-4, nbr, mask, xb)
        lhs = O.reg_value(g, 1.0, 2e-4, nbr, mask, xb + d)
        rhs = O.reg_value(g, 1.0, 2e-4, nbr, mask, xb) + (gr * d).sum() + 0.5 * (cu * d * d).sum()
        worst = min(worst, (rhs - lhs) / max(rhs, 1e-300))
    assert worst >= -1e-10


# ---------------------------------------------------------------- OS-LALM loop

def _subset_grad_py(g, M, m, y, w, x):
    """M A_m'(W(A_m x - y)) assembled from the oracle's projector (building block)."""
    cnt = O.nviews(g, m, M)
    p = O.fwd(g, x, m, M)
    p = M * w[m::M][:cnt] * (p - y[m::M][:cnt])
    return O.back(g, p, m, M)


def test_rho_one_is_os_sqs():
    """rho == 1 reduces OS-LALM to OS-SQS: iterate-identical to a separately
    written OS-SQS loop  x <- max(0, x - (M grad l_m(x) + grad R)/(D_L + D_R))."""
    g, y, w, mask = _small_problem()
    dl, S = O.sqs_denom(g, w, mask)
    M, K, beta, delta = 4, 3, 2.0 ** 10, 2e-4
    x0 = np.zeros(O.img_shape(g))
    x_lalm, log, _, _ = O.oslalm_run(g, y, w, dl, S, x0, M=M, mode="fixed", rho_fixed=1.0,
                                     beta=beta, delta=delta, nbr=8, n_iter=K)
    order = O.bit_reversal(M)
    x = x0.copy()
    for k in range(K):
        for j in range(M):
            G = _subset_grad_py(g, M, order[j], y, w, x)
            gr, cu = O.reg_grad(g, beta, delta, 8, S, x)
            x = np.where(S > 0, np.maximum(0.0, x - (G + gr) / np.where(S > 0, dl + cu, 1.0)), 0.0)
    assert np.abs(x - x_lalm).max() <= 1e-12 * np.abs(x).max()
    assert (log[:, 0] == 1.0).all()


def test_monotone_cost_M1_rho1():
    """M = 1, rho == 1 is a majorise-minimise SQS step, so Psi decreases monotonically (G19)."""
    g, y, w, mask = _small_problem()
    dl, S = O.sqs_denom(g, w, mask)
    beta, delta = 2.0 ** 12, 2e-4
    x = np.zeros(O.img_shape(g))
    costs = [O.cost(g, y, w, beta, delta, 8, S, x)]
    for it in range(200):
        x, _, _, _ = O.oslalm_run(g, y, w, dl, S, x, M=1, mode="fixed", rho_fixed=1.0,
                                  beta=beta, delta=delta, nbr=8, n_iter=1)
        costs.append(O.cost(g, y, w, beta, delta, 8, S, x))
    c = np.array(costs)
    assert (np.diff(c) <= 1e-12 * np.abs(c[:-1])).all()
    assert c[-1] < 0.2 * c[0]


@pytest.mark.parametrize("M,K", [(4, 6), (1, 150)])
def test_python_reimplementation_of_O7_continuation(M, K):
    """The oracle's loop (rho timing, xi, g-update, restart, counter) equals a separately
    written Python transcription of P:380-397 + P:495-516 (O7), log entry for log entry."""
    g, y, w, mask = _small_problem(seed=12)
    dl, S = O.sqs_denom(g, w, mask)
    beta, delta = 2.0 ** 11, 2e-4
    x0 = np.zeros(O.img_shape(g))
    xo, log, go, Go = O.oslalm_run(g, y, w, dl, S, x0, M=M, mode="continuation",
                                   beta=beta, delta=delta, nbr=8, n_iter=K, trailing=True)
    order = O.bit_reversal(M)
    Sm = S > 0
    x = x0.copy()
    G = _subset_grad_py(g, M, order[0], y, w, x)
    gsplit = G.copy()
    l = 0
    step = 0
    for k in range(K):
        for j in range(M):
            rho = 1.0 if l == 0 else max(math.pi / (l + 1) * math.sqrt(1 - (math.pi / (2 * l + 2)) ** 2), 1e-3)
            s = rho * G + (1 - rho) * gsplit
            gr, cu = O.reg_grad(g, beta, delta, 8, S, x)
            x = np.where(Sm, np.maximum(0.0, x - (s + gr) / np.where(Sm, rho * dl + cu, 1.0)), 0.0)
            Gp = _subset_grad_py(g, M, order[(j + 1) % M], y, w, x)
            xi = ((gsplit - Gp) * (Gp - G))[Sm].sum()
            gsplit = (rho * Gp + gsplit) / (1 + rho)
            G = Gp
            l = 0 if xi > 0 else l + 1
            assert log[step, 0] == pytest.approx(rho, rel=1e-12, abs=0)
            assert log[step, 1] == pytest.approx(xi, rel=1e-9, abs=1e-12 * abs(xi))
            assert log[step, 2] == (1.0 if xi > 0 else 0.0)
            step += 1
    assert np.abs(x - xo).max() <= 1e-10 * np.abs(x).max()
    assert np.abs(gsplit - go).max() <= 1e-10 * np.abs(gsplit).max()
    if M == 1:
        assert log[:, 2].sum() >= 1      # restarts fire at M = 1 on this problem (V7)


def _bruteforce_solution(g, y, w, S, beta, delta):
    """x_hat = argmin_{x >= 0 on S} 1/2||y - Ax||_W^2 + R(x): L-BFGS-B then projected Newton,
    with R and its derivatives written here from the pair list (independent of the oracle)."""
    A = _dense_A(g)
    Sm = S.reshape(-1) > 0
    As = A[:, Sm]
    W = w.reshape(-1); yv = y.reshape(-1)
    j, k, wt = _pairs(O.img_shape(g), 8)
    both = Sm[j] & Sm[k]
    pos = -np.ones(Sm.size, int); pos[Sm] = np.arange(Sm.sum())
    j, k, wt = pos[j[both]], pos[k[both]], wt[both]

    def f(xs):
        r = As @ xs - yv
        t = xs[j] - xs[k]
        a = np.abs(t) / delta
        val = 0.5 * (W * r * r).sum() + beta * (wt * delta * delta * (a - np.log1p(a))).sum()
        gd = As.T @ (W * r)
        ps = beta * wt * t / (1 + a)
        gd += np.bincount(j, ps, Sm.sum()) - np.bincount(k, ps, Sm.sum())
        return val, gd

    n = Sm.sum()
    res = scipy.optimize.minimize(f, np.full(n, 0.01), jac=True, method="L-BFGS-B",
                                  bounds=[(0, None)] * n, options=dict(maxiter=200000, maxfun=400000,
                                                                        ftol=0, gtol=1e-13, maxcor=50))
    xs = res.x
    H0 = As.T @ (W[:, None] * As)
    for it in range(60):
        val, gd = f(xs)
        t = xs[j] - xs[k]
        h2 = beta * wt / (1 + np.abs(t) / delta) ** 2
        H = H0.copy()
        np.add.at(H, (j, j), h2); np.add.at(H, (k, k), h2)
        np.add.at(H, (j, k), -h2); np.add.at(H, (k, j), -h2)
        free = ~((xs <= 0) & (gd > 0))
        step = np.zeros(n)
        step[free] = np.linalg.solve(H[np.ix_(free, free)], gd[free])
        a = 1.0
        while a > 1e-12:
            xn = np.maximum(0.0, xs - a * step)
            if f(xn)[0] <= val:
                break
            a *= 0.5
        xs = xn
    out = np.zeros(Sm.size); out[Sm] = xs
    kkt = np.where(xs > 0, np.abs(gd), np.maximum(0, -gd)).max()
    return out.reshape(O.img_shape(g)), kkt, f


def test_converges_to_bruteforce_minimiser_16x16():
    """OS-LALM M=1 with downward continuation converges to the brute-force minimiser (V5):
    relative error <= 1e-8 within 2500 iterations (dx 8 mm, 24 ch x 14 mm, 36 views,
    I0 = 1e4, beta = 2^16, delta = 2e-4, 8-nbr).  (With this phantom the error is 1.5e-6
    at 1500, 4e-8 at 2000 and ~1e-12 by 3500 iterations: linear convergence to x_hat.)"""
    g, y, w, mask = _small_problem()
    dl, S = O.sqs_denom(g, w, mask)
    beta, delta = 2.0 ** 16, 2e-4
    xhat, kkt, f = _bruteforce_solution(g, y, w, S, beta, delta)
    x = np.zeros(O.img_shape(g))
    x, log, _, _ = O.oslalm_run(g, y, w, dl, S, x, M=1, mode="continuation", beta=beta, delta=delta,
                                nbr=8, n_iter=2500)
    err = np.linalg.norm(x - xhat) / np.linalg.norm(xhat)
    assert kkt <= 1e-7
    assert err <= 1e-8, (err, kkt)
    assert (xhat == 0).sum() > 20          # the box constraint is active on part of S
    assert log[:, 2].sum() >= 1            # continuation restarted at least once


# ---------------------------------------------------------------- inner FISTA (NEXT-1)

def _inner_case(seed=21, beta=2.0 ** 10, nbr=8):
    g, y, w, mask = _small_problem()
    dl, S = O.sqs_denom(g, w, mask)
    rng = np.random.default_rng(seed)
    shape = O.img_shape(g)
    xk = rng.random(shape) * 0.02 * (S > 0)
    s = (rng.standard_normal(shape) * 0.5 * dl.max() * 1e-3) * (S > 0)
    return g, dl, S, xk, s, beta, 2e-4, nbr


def test_inner_fista_beta0_is_box_projection():
    """beta = 0: the inner problem is a D_L-weighted projection, solved exactly by one step:
    x = max(0, z), z = x_k - s / (rho D_L); further iterations stay there."""
    g, dl, S, xk, s, _, delta, nbr = _inner_case()
    rho = 0.3
    Sm = S > 0
    z = np.where(Sm, xk - s / np.where(Sm, rho * dl, 1.0), 0.0)
    for n in (1, 3):
        x = O.inner_fista(g, 0.0, delta, nbr, S, dl, rho, xk, s, n)
        assert np.abs(x - np.maximum(z, 0.0)).max() <= 1e-15 * max(1.0, np.abs(z).max())


def _inner_reference(g, dl, S, xk, s, beta, delta, rho):
    """High-accuracy solve of min_{x >= 0 on S} R(x) + rho/2 ||x - z||^2_{D_L} (L-BFGS-B, independent R)."""
    Sm = S.reshape(-1) > 0
    z = (xk - s / np.where(S > 0, rho * dl, 1.0)).reshape(-1)[Sm]
    D = dl.reshape(-1)[Sm]
    j, k, wt = _pairs(O.img_shape(g), 8)
    both = Sm[j] & Sm[k]
    pos = -np.ones(Sm.size, int); pos[Sm] = np.arange(Sm.sum())
    j, k, wt = pos[j[both]], pos[k[both]], wt[both]

    def f(xs):
        t = xs[j] - xs[k]
        a = np.abs(t) / delta
        val = beta * (wt * delta * delta * (a - np.log1p(a))).sum() + 0.5 * rho * (D * (xs - z) ** 2).sum()
        ps = beta * wt * t / (1 + a)
        gd = np.bincount(j, ps, Sm.sum()) - np.bincount(k, ps, Sm.sum()) + rho * D * (xs - z)
        return val, gd

    res = scipy.optimize.minimize(f, np.maximum(z, 0), jac=True, method="L-BFGS-B", bounds=[(0, None)] * Sm.sum(),
                                  options=dict(maxiter=100000, maxfun=200000, ftol=0, gtol=1e-16, maxcor=50))
    out = np.zeros(Sm.size); out[Sm] = res.x
    return out.reshape(O.img_shape(g))


def test_inner_fista_converges_to_inner_minimiser():
    """n -> large: FISTA reaches the exact inner minimiser."""
    g, dl, S, xk, s, beta, delta, nbr = _inner_case()
    rho = 0.5
    ref = _inner_reference(g, dl, S, xk, s, beta, delta, rho)
    x = O.inner_fista(g, beta, delta, nbr, S, dl, rho, xk, s, 3000)
    assert np.linalg.norm(x - ref) <= 1e-7 * np.linalg.norm(ref)
    # more iterations never hurt much, few iterations are already close (warm start)
    x5 = O.inner_fista(g, beta, delta, nbr, S, dl, rho, xk, s, 5)
    assert np.linalg.norm(x5 - ref) < np.linalg.norm(xk - ref)


def test_inner_fista_warm_start_at_solution_is_fixed():
    """Warm start at the inner solution (same z) is a fixed point."""
    g, dl, S, xk, s, beta, delta, nbr = _inner_case()
    rho = 0.5
    xs = O.inner_fista(g, beta, delta, nbr, S, dl, rho, xk, s, 4000)
    Sm = S > 0
    z = np.where(Sm, xk - s / np.where(Sm, rho * dl, 1.0), 0.0)
    s2 = np.where(Sm, rho * dl * (xs - z), 0.0)          # keeps z unchanged for x_k = xs
    x = O.inner_fista(g, beta, delta, nbr, S, dl, rho, xs, s2, 5)
    assert np.abs(x - xs).max() <= 1e-10 * np.abs(xs).max()


def test_oslalm_fista_inner_converges_to_bruteforce():
    """OS-LALM with n = 3 inner FISTA iterations (M = 1, continuation) has the same fixed point:
    the brute-force minimiser of the 16x16 problem."""
    g, y, w, mask = _small_problem()
    dl, S = O.sqs_denom(g, w, mask)
    beta, delta = 2.0 ** 16, 2e-4
    xhat, kkt, f = _bruteforce_solution(g, y, w, S, beta, delta)
    x = np.zeros(O.img_shape(g))
    x, log, _, _ = O.oslalm_run(g, y, w, dl, S, x, M=1, mode="continuation", beta=beta, delta=delta,
                                nbr=8, n_iter=3000, inner="fista", n_inner=3)
    err = np.linalg.norm(x - xhat) / np.linalg.norm(xhat)
    assert err <= 1e-6, err
