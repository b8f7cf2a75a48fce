"""GPU model selection along the λ path against the oracle:
ν, OLS-de-biased rss, GCV, e-BIC per point, the selected index, and the max-active cap."""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import cuda_ok

pytestmark = pytest.mark.gpu

if cuda_ok():
    from paper_2006_03970_b200 import Problem
    from paper_2006_03970_b200.path import lambda_grid, solve_path


def oracle_path(A, b, alpha, cs, max_active=None):
    """The oracle's warm-started path (σ carried, R38) with the criteria at every point."""
    ls, res = oracle.solve_path(A, b, alpha, cs, max_active=max_active)
    pts = []
    for (l1, l2), (x, _, st) in zip(ls, res):
        r, nu, rss, gcv, ebic, xdb = oracle.model_select(A, b, x, l2)
        pts.append({"r": r, "nu": nu, "rss": rss, "gcv": gcv, "ebic": ebic, "xdb": xdb, "active": st["active"]})
    return pts


def test_path_selection_matches_oracle():
    cfg = synth.scaled(synth.CONFIGS["cfg2"], n=20_000)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    cs = lambda_grid(30)
    ref = oracle_path(A, b, cfg.alpha, cs, max_active=100)
    with Problem(A, b) as P:
        pts, best = solve_path(P, cfg.alpha, cs, max_active=100, debias=True)
    assert len(pts) == len(ref)
    for p, q in zip(pts, ref):
        cr = p["criteria"]
        assert cr["active"] == q["r"] == p["stats"]["active"]
        assert cr["nu"] == pytest.approx(q["nu"], rel=1e-9, abs=1e-12)
        assert cr["rss"] == pytest.approx(q["rss"], rel=1e-8)
        assert cr["gcv"] == pytest.approx(q["gcv"], rel=1e-8)
        assert cr["ebic"] == pytest.approx(q["ebic"], rel=1e-8, abs=1e-10)
        assert cr["ols_ok"] == 1
        np.testing.assert_allclose(p["x_debiased"], q["xdb"], rtol=1e-7, atol=1e-9 * np.abs(q["xdb"]).max(initial=1))
    for key in ("gcv", "ebic"):
        assert best[key] == int(np.argmin([q[key] for q in ref]))


def test_dof_push_through_branch():
    """r ≥ m: ν = m − λ2‖L⁻¹‖_F² of K + λ2 I, K = A_J A_Jᵀ (push-through identity) vs the oracle's
    r × r computation; OLS is undefined there (ols_ok = 0, rss NaN)."""
    cfg = synth.Config("dof", 40, 300, synth.IID_STD, 5, 1.0, 2.0, 5.0, 0.3, (0.02,), 71)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    lm = float(np.max(np.abs(oracle.aty(A, b)))) / cfg.alpha
    l1, l2 = 0.02 * cfg.alpha * lm, 0.02 * (1 - cfg.alpha) * lm
    with Problem(A, b) as P:
        x, st = P.solve(l1, l2, 5e-3, 1e-8)
        crit, _ = P.model_select(l2)
    J = np.nonzero(x)[0]
    assert len(J) >= cfg.m
    assert crit["nu"] == pytest.approx(oracle.dof(A, J, l2), rel=1e-9)
    assert crit["ols_ok"] == 0 and np.isnan(crit["rss"])


def test_empty_support_criteria():
    cfg = synth.scaled(synth.CONFIGS["cfg1"], n=300)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    with Problem(A, b) as P:
        g = P.lambda_max_l1
        x, st = P.solve(g, 0.1 * g, 5e-3, 1e-6)
        crit, xdb = P.model_select(0.1 * g, debias=True)
    assert crit["active"] == 0 and crit["nu"] == 0.0 and np.all(xdb == 0)
    assert crit["rss"] == pytest.approx(float(b @ b), rel=1e-13)
    assert crit["gcv"] == pytest.approx(float(b @ b) / cfg.m, rel=1e-13)
