"""Pins for the oracle's Barzilai-Borwein scaling (NEXT-2).

PAPER.md P:539 and supplement P:1472-1492 (eqs. secant_eq, scale_factor_alpha_k): the SQS
Hessian L_diag is replaced by H_k = alpha_k L_diag, alpha_k fitting y_k ~ H_k s_k in the
P = L_diag^{-1} weighted least-squares sense with alpha <= 1.  OS reading B-BB:
k counts outer iterations, grad l(x^k) ~ mean of the iteration's M subset gradients; with
M = 1 that mean is the exact gradient at x^k, so y_k = A'WA s_k and alpha_{k+1} is the
Rayleigh quotient ||A s_k||_W^2 / ||s_k||_{L_diag}^2 — computed here with the oracle's
forward projector in the data domain, not with the secant formula the oracle uses.
"""
import numpy as np

import oracle as O
from tests.test_oracle_algorithm import _bruteforce_solution, _small_problem


def _run(g, y, w, dl, S, n_iter, **kw):
    a = np.zeros(n_iter)
    x, log, gs, Gs = O.oslalm_run(g, y, w, dl, S, np.zeros(O.img_shape(g)), n_iter=n_iter, alpha_out=a, **kw)
    return x, log, a


def test_bb_alpha_min_one_is_plain_oslalm():
    """alpha clipped to [1, 1] gives H_k = L_diag: iterate-identical to OS-LALM without BB."""
    g, y, w, mask = _small_problem(seed=5)
    dl, S = O.sqs_denom(g, w, mask)
    kw = dict(M=4, beta=2.0 ** 11, delta=2e-4, nbr=8)
    x0, log0, _ = _run(g, y, w, dl, S, 6, **kw)
    x1, log1, a1 = _run(g, y, w, dl, S, 6, bb=True, alpha_min=1.0, **kw)
    assert np.array_equal(x0, x1) and np.array_equal(log0, log1)
    assert (a1 == 1.0).all()


def test_bb_alpha_is_data_domain_rayleigh_quotient_M1():
    """M = 1: alpha used in iteration k+1 = clip(||A s||_W^2 / (s' D_L s)), s = x^k - x^{k-1};
    and 0 < alpha <= 1 because D_L majorises A'WA (SQS inequality)."""
    g, y, w, mask = _small_problem(seed=7)
    dl, S = O.sqs_denom(g, w, mask)
    kw = dict(M=1, beta=2.0 ** 12, delta=2e-4, nbr=8, bb=True)
    K = 6
    xs = [np.zeros(O.img_shape(g))]
    for k in range(1, K + 1):
        x, _, _ = _run(g, y, w, dl, S, k, **kw)
        xs.append(x)
    _, _, a = _run(g, y, w, dl, S, K, **kw)
    assert a[0] == 1.0 and a[1] == 1.0          # no secant pair before iteration 3
    ww = np.reshape(w, O.sino_shape(g, g["na"]))
    for k in range(2, K):                        # alpha[k] is used in iteration k + 1
        s = xs[k] - xs[k - 1]
        As = O.fwd(g, s)
        rq = float((ww * As * As).sum() / (dl * s * s)[S > 0].sum())
        assert 0.0 < rq <= 1.0 + 1e-12
        assert abs(a[k] - min(1.0, rq)) <= 1e-9 * rq, (k, a[k], rq)


def test_bb_converges_to_bruteforce_minimiser_16x16():
    """BB changes the metric, not the fixed point: with rho = 1 (OS-SQS, M = 1) the scaled
    iteration converges to the brute-force minimiser of the 16x16 problem (V5) and much faster
    than the plain SQS iteration (the acceleration P:1492 reports); with continuation it also
    converges to the same point."""
    g, y, w, mask = _small_problem()
    dl, S = O.sqs_denom(g, w, mask)
    beta, delta = 2.0 ** 16, 2e-4
    xhat, kkt, _ = _bruteforce_solution(g, y, w, S, beta, delta)
    assert kkt <= 1e-7
    err = lambda x: np.linalg.norm(x - xhat) / np.linalg.norm(xhat)
    kw = dict(M=1, beta=beta, delta=delta, nbr=8)
    x_bb, _, a = _run(g, y, w, dl, S, 3000, mode="fixed", rho_fixed=1.0, bb=True, **kw)
    x_sqs, _, _ = _run(g, y, w, dl, S, 3000, mode="fixed", rho_fixed=1.0, **kw)
    assert err(x_bb) <= 1e-5 and err(x_sqs) >= 1e-2, (err(x_bb), err(x_sqs))
    assert (a[2:] < 1.0).all() and (a > 0).all()
    x_c, _, _ = _run(g, y, w, dl, S, 4000, bb=True, **kw)
    assert err(x_c) <= 1e-6, err(x_c)


def test_bb_os_bookkeeping_matches_python_transcription_M4():
    """OS reading B-BB: alpha_k = clip(y's / s'D_L s, alpha_min, 1) with
    y = gbar_k - gbar_{k-1} (mean subset gradients of iterations k, k-1) and s = xbar_k -
    xbar_{k-1} (mean of the inner iterates those gradients were taken at); alpha_k is used
    in iteration k + 1.  A separately written Python loop (plain SQS inner step, fixed rho)
    must reproduce the oracle's alpha sequence and image."""
    from tests.test_oracle_algorithm import _subset_grad_py
    g, y, w, mask = _small_problem(seed=3)
    dl, S = O.sqs_denom(g, w, mask)
    beta, delta, M, K, rho, amin = 2.0 ** 11, 2e-4, 4, 7, 0.5, 1e-6
    x0 = np.zeros(O.img_shape(g))
    a_or = np.zeros(K)
    xo, _, _, _ = O.oslalm_run(g, y, w, dl, S, x0, M=M, mode="fixed", rho_fixed=rho, beta=beta, delta=delta,
                               nbr=8, n_iter=K, trailing=True, bb=True, alpha_min=amin, alpha_out=a_or)
    order = O.bit_reversal(M)
    Sm = S > 0
    x = x0.copy()
    G = _subset_grad_py(g, M, order[0], y, w, x)
    gs = G.copy()
    alpha, alphas = 1.0, []
    gbar_prev = xbar_prev = None
    for k in range(1, K + 1):
        alphas.append(alpha)
        gbar = np.zeros_like(x)
        xbar = np.zeros_like(x)
        for j in range(M):
            s = rho * G + (1 - rho) * gs
            gr, cu = O.reg_grad(g, beta, delta, 8, S, x)
            x = np.where(Sm, np.maximum(0.0, x - (s + gr) / np.where(Sm, rho * alpha * dl + cu, 1.0)), 0.0)
            Gp = _subset_grad_py(g, M, order[(j + 1) % M], y, w, x)
            gs = (rho * Gp + gs) / (1 + rho)
            G = Gp
            gbar += G / M
            xbar += x / M
        if k >= 2:
            sv = (xbar - xbar_prev)[Sm]
            num = ((gbar - gbar_prev)[Sm] * sv).sum()
            den = (dl[Sm] * sv * sv).sum()
            alpha = min(1.0, max(amin, num / den if den > 0 else 1.0))
        gbar_prev, xbar_prev = gbar, xbar
    assert np.allclose(alphas, a_or, rtol=1e-9, atol=0), (alphas, a_or)
    assert (np.array(alphas[2:]) < 1.0).any()
    assert np.abs(x - xo).max() <= 1e-9 * np.abs(x).max()
