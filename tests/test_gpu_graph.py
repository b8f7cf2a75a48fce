"""Graph mode (device-resident control, nested conditional WHILE graph) against the host-driven
mode: both take the same decisions with the same IEEE operations on the same values and launch
the same work decompositions (DirGeo), so x and every statistic must be bitwise identical.
The host-driven mode is itself held to the oracle by test_gpu_solve / test_gpu_fullsize."""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import compare_to_oracle, cuda_ok

pytestmark = pytest.mark.gpu

if cuda_ok():
    from paper_2006_03970_b200 import Problem

SAME = ["status", "outer_iters", "newton_iters", "psi_evals", "backtracks", "aty_passes", "branch_steps",
        "line_search_stalled", "active", "res_kkt1", "res_kkt3", "primal_obj", "dual_obj", "gap", "sigma_final"]

_seen = {"backtracks": 0, "branch": [0, 0, 0], "stalled": 0, "not_converged": 0}


def both(P, l1, l2, sigma0=5e-3, tol=1e-6, x0=None):
    P.set_option("small", 0)  # the one-CTA path (k_small_solve) would serve both modes at cfg1 size
    P.set_option("graph", 0)
    xh, sh = P.solve(l1, l2, sigma0, tol, x0=x0)
    P.set_option("graph", 1)
    xg, sg = P.solve(l1, l2, sigma0, tol, x0=x0)
    assert np.array_equal(xh, xg), np.max(np.abs(xh - xg))
    for k in SAME:
        a, b = sh[k], sg[k]
        same = (a == b) or (isinstance(a, float) and np.isnan(a) and np.isnan(b))
        assert same, (k, a, b, sh, sg)
    _seen["backtracks"] += sg["backtracks"]
    for i in range(3):
        _seen["branch"][i] += sg["branch_steps"][i]
    _seen["stalled"] += sg["line_search_stalled"]
    _seen["not_converged"] += sg["status"] == 1
    return xg, sg


def lambdas(cfg, lm, c):
    lmax = lm / cfg.alpha
    return c * cfg.alpha * lmax, c * (1 - cfg.alpha) * lmax


def test_graph_cfg1_all_c():
    cfg = synth.CONFIGS["cfg1"]
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    with Problem(A, b) as P:
        assert P.info("graph") == 1  # default mode
        lm = P.lambda_max_l1
        for c in cfg.cs:
            l1, l2 = lambdas(cfg, lm, c)
            both(P, l1, l2)


def test_graph_cfg2_path_warm():
    """BASELINE configs[1] shape, warm-started along the path (Table D.4 grid)."""
    cfg = synth.CONFIGS["cfg2"]
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    with Problem(A, b) as P:
        lm = P.lambda_max_l1
        xprev = None
        for c in cfg.cs[:5]:
            l1, l2 = lambdas(cfg, lm, c)
            xprev, st = both(P, l1, l2, x0=xprev)
            assert st["status"] == 0


def test_graph_branches_and_options():
    """r ≥ m (Eq. (18)) and r < m (Eq. (19)) steps, lasso, x = 0 above λmax, capped loops,
    a strict Armijo constant (μ = 0.49) to force backtracking, max_backtracks = 0 (R30)."""
    cfg = synth.scaled(synth.CONFIGS["cfg3"], n=3000)
    A = synth.design(cfg)[:, :]
    b, _ = synth.response(cfg)
    Asm = np.ascontiguousarray(A[:, :])
    # small m so that r ≥ m happens at small λ
    cfg_s = synth.scaled(synth.CONFIGS["cfg1"], n=1500)
    As = synth.design(cfg_s)
    bs, _ = synth.response(cfg_s)
    with Problem(Asm, b) as P:
        lm = P.lambda_max_l1
        both(P, 0.3 * lm, 0.1 * lm)
        both(P, 0.05 * lm, 0.01 * lm)
        both(P, 0.1 * lm, 0.0)                    # lasso
        both(P, lm, 0.3 * lm)                     # x = 0
        P.set_option("max_outer", 2)
        both(P, 0.05 * lm, 0.01 * lm)             # not converged
        P.set_option("max_outer", 100)
        P.set_option("mu", 0.49)
        both(P, 0.05 * lm, 0.01 * lm, sigma0=1.0)
        both(P, 0.2 * lm, 0.05 * lm, sigma0=20.0)
        P.set_option("max_backtracks", 0)
        both(P, 0.05 * lm, 0.01 * lm, sigma0=20.0)
    with Problem(As, bs) as P:
        lm = P.lambda_max_l1
        for c in (0.5, 0.05, 0.005, 0.001):
            both(P, c * lm, 0.2 * c * lm, sigma0=1.0)
        P.set_option("mu", 0.49)
        both(P, 0.001 * lm, 0.0002 * lm, sigma0=50.0)
    assert _seen["branch"][1] > 0 and _seen["branch"][2] > 0 and _seen["branch"][0] > 0, _seen
    assert _seen["backtracks"] > 0, _seen
    assert _seen["not_converged"] > 0, _seen


def test_graph_matches_oracle_cfg1():
    """Graph mode directly against the oracle (same bar as test_gpu_solve)."""
    from gpu_util import solution_parity
    cfg = synth.CONFIGS["cfg1"]
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    lm = float(np.max(np.abs(oracle.aty(A, b))))
    with Problem(A, b) as P:
        P.set_option("small", 0)
        for c in cfg.cs:
            l1, l2 = lambdas(cfg, lm, c)
            xc, _, stc, _ = oracle.solve(A, b, l1, l2, sigma0=5e-3, tol=1e-6)
            xg, stg = P.solve(l1, l2, 5e-3, 1e-6)
            Fg = oracle.primal_obj(A, b, xg, l1, l2)
            Fc = oracle.primal_obj(A, b, xc, l1, l2)
            assert solution_parity(xg, xc, Fg, Fc)["ok"]
            assert stg["outer_iters"] == stc["outer_iters"]


def test_graph_rebuild_after_cluster_change():
    cfg = synth.CONFIGS["cfg1"]
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    with Problem(A, b) as P:
        P.set_option("small", 0)
        lm = P.lambda_max_l1
        x1, s1 = P.solve(0.1 * lm, 0.05 * lm)
        P.set_option("cluster_size", 8)
        x2, s2 = P.solve(0.1 * lm, 0.05 * lm)
        assert s2["status"] == 0
        np.testing.assert_allclose(x2, x1, rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_gram_kernel_options_agree(mode):
    """Option gram_sk selects the K3 kernel (0: k_gram_fused for both branches, 1: fused for SMW and
    k_gram_sk for m × m — the default —, 2: k_gram_sk for both); graph ≡ host bitwise in every mode and
    every mode meets the oracle (cfg3 recipe at n = 2e4: SMW steps at c = 0.3, m × m at c = 0.05)."""
    cfg = synth.scaled(synth.CONFIGS["cfg3"], n=20_000)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    lm = float(np.max(np.abs(oracle.aty(A, b)))) / cfg.alpha
    seen = np.zeros(4, dtype=int)
    for c in (0.3, 0.05):
        l1, l2 = c * cfg.alpha * lm, c * (1 - cfg.alpha) * lm
        out = {}
        for graph in (1, 0):
            with Problem(A, b) as P:
                P.set_option("gram_sk", mode)
                P.set_option("graph", graph)
                out[graph] = P.solve(l1, l2, cfg.sigma0, cfg.tol)
        assert np.array_equal(out[0][0], out[1][0])
        for k in ("outer_iters", "newton_iters", "branch_steps", "res_kkt1", "res_kkt3", "primal_obj", "dual_obj"):
            assert out[0][1][k] == out[1][1][k], k
        seen += np.array(out[1][1]["branch_steps"])

        def gpu(s0, tol, x0, mode=mode, l1=l1, l2=l2):
            with Problem(A, b) as P:
                P.set_option("gram_sk", mode)
                return P.solve(l1, l2, s0, tol, x0=x0)

        compare_to_oracle(A, b, l1, l2, gpu, sigma0=cfg.sigma0, tol=cfg.tol, label=("gram_sk", mode, c))
    assert seen[1] > 0 and seen[2] > 0
