"""K6 (conjugate-gradient Newton direction; reading R32) against
the oracle: the direction through the C-ABI hook vs oracle.cg_direction and the exact branches,
iteration-level agreement at a fixed iteration cap, and whole solves with the CG strategy vs the
oracle run with the same strategy (and vs the exact branches)."""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import cuda_ok, dev, empty, host, solution_parity

pytestmark = pytest.mark.gpu

if cuda_ok():
    import torch
    from paper_2006_03970_b200 import Problem


def inputs(kind, m, n, seed):
    cfg = synth.Config("cg", m, n, kind, 5, 1.0, 2.0, 5.0, 0.7, (0.5,), seed)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    return A, b


def hook(P, J, g, kappa):
    m = len(g)
    dJ, dg, dd = dev(J.astype(np.int32)), dev(g), empty(m)
    gd, br = P.newton_direction(dJ.data_ptr() if len(J) else 0, len(J), dg.data_ptr(), kappa, dd.data_ptr())
    torch.cuda.synchronize()
    return host(dd, m), gd, br


@pytest.mark.parametrize("kind,m,n,r,kappa", [
    (synth.IID_STD, 50, 600, 400, 0.5),       # r ≫ m
    (synth.IID_STD, 100, 400, 30, 2e-3),      # r < m
    (synth.AR1_STD, 500, 12000, 10000, 5e-3),  # cfg2-like early iteration (r = 20 m)
    (synth.IID_STD, 800, 5000, 4000, 1e-2),   # m = 800 (MR = 25)
    (synth.IID_UNIT_L2, 7, 40, 3, 3.0),       # tiny m, one warp-row
])
def test_cg_direction_parity(kind, m, n, r, kappa):
    seed = 51
    A, b = inputs(kind, m, n, seed)
    J = np.sort((np.argsort(synth.uniforms(seed, 7, n))[:r]).astype(np.int64))
    g = synth.normals(seed, 8, m) * 3
    d_exact, _ = oracle.newton_direction(A, J, g, kappa)
    d_orc, it_orc = oracle.cg_direction(A, J, g, kappa, tol=1e-10)
    with Problem(A, b) as P:
        P.set_option("cg_ratio", 1e-9)
        P.set_option("cg_tol", 1e-10)
        d, gd, br = hook(P, J, g, kappa)
    assert br == 3
    scale = np.linalg.norm(d_exact)
    # both stop at ‖Vd + g‖ ≤ 1e-10‖g‖; V's condition number bounds the error in d
    AJ = A[J].T
    V = np.eye(m) + kappa * AJ @ AJ.T
    resid = np.linalg.norm(V @ d + g) / np.linalg.norm(g)
    assert resid <= 2e-10, resid
    assert np.linalg.norm(d - d_exact) <= 1e-7 * scale
    assert np.linalg.norm(d - d_orc) <= 1e-7 * scale
    assert gd == pytest.approx(g @ d, rel=1e-12) and gd < 0


@pytest.mark.parametrize("maxit", [1, 2, 5])
def test_cg_fixed_iterations_match_oracle(maxit):
    """With the iteration cap binding, GPU and oracle run the same Krylov iterates: equal up to rounding."""
    m, n, r, kappa, seed = 120, 900, 700, 0.8, 52
    A, b = inputs(synth.IID_STD, m, n, seed)
    J = np.sort((np.argsort(synth.uniforms(seed, 7, n))[:r]).astype(np.int64))
    g = synth.normals(seed, 8, m)
    d_orc, it = oracle.cg_direction(A, J, g, kappa, tol=1e-30, maxit=maxit)
    assert it == maxit
    with Problem(A, b) as P:
        P.set_option("cg_ratio", 1e-9)
        P.set_option("cg_maxit", maxit)
        d, gd, br = hook(P, J, g, kappa)
    assert br == 3
    assert np.max(np.abs(d - d_orc)) <= 1e-12 * np.max(np.abs(d_orc))
    assert gd < 0


def test_cg_strategy_rule():
    """Default: the paper's rule (min(m, r) > 1e4) never selects CG at m ≤ 1024; cg_ratio opts in."""
    m, n, seed = 60, 500, 53
    A, b = inputs(synth.IID_STD, m, n, seed)
    J = np.arange(0, 300, dtype=np.int64)
    g = synth.normals(seed, 8, m)
    with Problem(A, b) as P:
        _, _, br = hook(P, J, g, 0.3)
        assert br == 2
        P.set_option("cg_ratio", 4.0)  # CG iff r > 4m = 240
        _, _, br = hook(P, J, g, 0.3)
        assert br == 3
        _, _, br = hook(P, J[:200], g, 0.3)
        assert br == 2
        P.set_option("cg_ratio", 0.0)
        P.set_option("cg_threshold", 50)  # min(m, r) = 60 > 50
        _, _, br = hook(P, J, g, 0.3)
        assert br == 3


@pytest.mark.parametrize("name,n,ratio", [("cfg1", None, 1e-9), ("cfg3", 20_000, 2.0), ("cfg2", 30_000, 2.0)])
def test_solve_with_cg_matches_oracle(name, n, ratio):
    """Whole solves with the CG strategy vs the oracle with the same strategy and vs the exact branches."""
    cfg = synth.CONFIGS[name] if n is None else synth.scaled(synth.CONFIGS[name], n=n)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    lm = float(np.max(np.abs(oracle.aty(A, b)))) / cfg.alpha
    cs = cfg.cs if not cfg.path else (0.5, 0.2)
    with Problem(A, b) as P:
        for c in cs:
            l1, l2 = c * cfg.alpha * lm, c * (1 - cfg.alpha) * lm
            xe, se = P.solve(l1, l2, cfg.sigma0, cfg.tol)
            P.set_option("cg_ratio", ratio)
            xg, sg = P.solve(l1, l2, cfg.sigma0, cfg.tol)
            P.set_option("cg_ratio", 0.0)
            xc, _, sc, _ = oracle.solve(A, b, l1, l2, sigma0=cfg.sigma0, tol=cfg.tol, cg_ratio=ratio)
            assert sg["status"] == 0 and sc["status"] == 0, (sg, sc)
            Fg = oracle.primal_obj(A, b, xg, l1, l2)
            Fc = oracle.primal_obj(A, b, xc, l1, l2)
            Fe = oracle.primal_obj(A, b, xe, l1, l2)
            assert solution_parity(xg, xc, Fg, Fc)["ok"], (c, sg, sc)
            assert solution_parity(xg, xe, Fg, Fe)["ok"], (c, sg, se)
            assert sg["outer_iters"] == sc["outer_iters"]
            assert abs(sg["newton_iters"] - sc["newton_iters"]) <= 1
            if ratio < 1e-6:
                assert sg["branch_steps"][3] == sg["newton_iters"] - sg["branch_steps"][0]
            assert sg["branch_steps"][3] == sc["branch_steps"][3] or abs(sg["newton_iters"] - sc["newton_iters"]) <= 1
            if sg["branch_steps"][3]:
                assert sg["cg_iters"] >= sg["branch_steps"][3]


def test_cg_graph_equals_host():
    cfg = synth.scaled(synth.CONFIGS["cfg2"], n=20_000)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    lm = float(np.max(np.abs(oracle.aty(A, b)))) / cfg.alpha
    with Problem(A, b) as P:
        P.set_option("cg_ratio", 1.5)
        for c in (0.3, 0.1):
            l1, l2 = c * cfg.alpha * lm, c * (1 - cfg.alpha) * lm
            P.set_option("graph", 0)
            xh, sh = P.solve(l1, l2, cfg.sigma0, cfg.tol)
            P.set_option("graph", 1)
            xg, sg = P.solve(l1, l2, cfg.sigma0, cfg.tol)
            assert np.array_equal(xh, xg)
            for k in ("outer_iters", "newton_iters", "branch_steps", "cg_iters", "backtracks", "res_kkt1",
                      "res_kkt3", "primal_obj"):
                assert sh[k] == sg[k], (k, sh[k], sg[k])


def test_cg_options_after_graph_build():
    """cg_tol / cg_maxit set after the handle's graph exists still reach the CG kernel (the graph is
    rebuilt): graph ≡ host with a truncated CG (R32)."""
    cfg = synth.scaled(synth.CONFIGS["cfg2"], n=20_000)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    lm = float(np.max(np.abs(oracle.aty(A, b)))) / cfg.alpha
    l1, l2 = 0.2 * cfg.alpha * lm, 0.2 * (1 - cfg.alpha) * lm
    with Problem(A, b) as P:
        P.set_option("cg_ratio", 1e-9)
        P.set_option("graph", 1)
        _, s0 = P.solve(l1, l2, cfg.sigma0, cfg.tol)  # graph built with the default cg options
        P.set_option("cg_maxit", 3)
        P.set_option("cg_tol", 1e-6)
        xg, sg = P.solve(l1, l2, cfg.sigma0, cfg.tol)
        P.set_option("graph", 0)
        xh, sh = P.solve(l1, l2, cfg.sigma0, cfg.tol)
        assert np.array_equal(xh, xg)
        assert sg["cg_iters"] == sh["cg_iters"] and sg["newton_iters"] == sh["newton_iters"]
        assert sg["branch_steps"][3] > 0
        assert sg["cg_iters"] <= 3 * sg["branch_steps"][3] < s0["cg_iters"]
