"""Pins for the oracle's adaptive inner tolerance (option inner_tol_mode = 1; "inner_tol at
outer iteration k is max(outer_tol, 0.1·res(kkt3) at iteration k)"; reading R37: res(kkt3) of
Eq. (20) at the point outer iteration k starts from, i.e. (x_k, y_k) with P = prox(x_k − σ_kAᵀy_k)).

The schedule is recomputed here in numpy from the iterates the oracle returns when stopped after
k outer iterations (x_k, y_k; σ_k = σ0·5^k), and checked against the Newton trace of outer
iteration k: every step taken had res1 > tol_in, and the inner loop ended at res1 ≤ tol_in.
The minimiser itself does not depend on the schedule (the outer stop still needs res1, res3 ≤ tol):
coordinate descent and the KKT inclusion pin it."""
import numpy as np
import pytest

import oracle
import synth


def soft(t, thr):
    return np.sign(t) * np.maximum(np.abs(t) - thr, 0.0)


def case(name="cfg1", c=0.2):
    cfg = synth.CONFIGS[name]
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    lm = float(np.max(np.abs(oracle.aty(A, b)))) / cfg.alpha
    return cfg, A, b, c * cfg.alpha * lm, c * (1 - cfg.alpha) * lm


@pytest.mark.parametrize("c", [0.5, 0.2, 0.1])
def test_schedule_against_trace(c):
    cfg, A, b, l1, l2 = case(c=c)
    kw = dict(sigma0=cfg.sigma0, tol=cfg.tol, inner_tol_mode=1)
    _, _, full, _ = oracle.solve(A, b, l1, l2, **kw)
    _, _, plain, _ = oracle.solve(A, b, l1, l2, sigma0=cfg.sigma0, tol=cfg.tol)
    assert full["status"] == 0
    for k in range(1, full["outer_iters"]):
        xk, yk, sk, _ = oracle.solve(A, b, l1, l2, max_outer=k, **kw)
        sigma = cfg.sigma0 * 5.0 ** k
        w = A @ yk  # (n, m) @ (m,) = Aᵀy
        P = soft(xk - sigma * w, sigma * l1) / (1 + sigma * l2)
        z = (xk - P) / sigma - w
        res3 = (np.linalg.norm(xk - P) / sigma) / (1 + np.linalg.norm(yk) + np.linalg.norm(z))
        tol_in = max(cfg.tol, 0.1 * res3)
        _, _, s2, tr = oracle.solve(A, b, l1, l2, max_outer=k + 1, trace_cap=10_000, **kw)
        steps = [t for t in tr if t["outer"] == k]
        assert all(t["res1"] > tol_in * (1 - 1e-9) for t in steps), k
        assert s2["res_kkt1"] <= tol_in * (1 + 1e-9), k
    assert full["newton_iters"] <= plain["newton_iters"]
    assert full["outer_iters"] == plain["outer_iters"] or abs(full["outer_iters"] - plain["outer_iters"]) <= 1


def test_same_minimiser_and_kkt():
    for name, c in (("cfg1", 0.3), ("cfg1", 0.1)):
        cfg, A, b, l1, l2 = case(name, c)
        x0, _, s0, _ = oracle.solve(A, b, l1, l2, sigma0=cfg.sigma0, tol=1e-10)
        x1, _, s1, _ = oracle.solve(A, b, l1, l2, sigma0=cfg.sigma0, tol=1e-10, inner_tol_mode=1)
        assert s0["status"] == 0 and s1["status"] == 0
        g = float(np.max(np.abs(oracle.aty(A, b))))
        assert oracle.kkt_violation(A, b, x1, l1, l2) <= 1e-8 * g
        assert np.max(np.abs(x1 - x0)) <= 1e-7 * np.max(np.abs(x0))
        assert s1["newton_iters"] < s0["newton_iters"]


def test_cold_start_first_outer_is_unchanged():
    """At x0 = 0, y0 = 0: P = 0 so res3 = 0 and tol_in = tol — the λ1 ≥ λmax case still takes
    exactly one Newton step."""
    cfg = synth.CONFIGS["cfg1"]
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    g = float(np.max(np.abs(oracle.aty(A, b))))
    x, y, st, _ = oracle.solve(A, b, g, 0.3 * g, inner_tol_mode=1)
    assert np.all(x == 0) and st["newton_iters"] == 1 and st["outer_iters"] == 1
