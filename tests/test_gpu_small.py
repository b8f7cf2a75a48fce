"""The single-launch solves for small problems (m ≤ 64, n ≤ 1024; Algorithm 1):
the 16-CTA cluster kernel k_small_cl (A resident in distributed shared memory; the default) and the
one-CTA kernel k_small_solve (option small_cluster = 0), each against the oracle — parity with the CPU oracle at BASELINE tolerances and the same iteration counts as the
oracle and the multi-kernel graph path, across shapes, both Newton branches (Eq. (18)/(19)), warm
starts, the oracle-free pins (x = 0 above λmax after one Newton step, warm start at the solution),
Lasso (λ2 = 0), the adaptive inner tolerance (R37), the factor retry (R36) and the iteration cap."""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import cuda_ok, solution_parity

pytestmark = pytest.mark.gpu

if cuda_ok():
    from paper_2006_03970_b200 import Problem

SHAPES = [  # (kind, m, n, alpha, seed): tiny / ragged (odd m·n: the TMA tail) / largest eligible shapes
    (synth.IID_UNIT_L2, 50, 1000, 0.7, 1),
    (synth.IID_STD, 2, 1, 0.5, 31),
    (synth.IID_STD, 7, 41, 0.5, 32),
    (synth.IID_STD, 33, 501, 0.3, 33),
    (synth.AR1_STD, 64, 1024, 0.7, 34),
    (synth.IID_STD, 64, 65, 0.5, 35),
    (synth.IID_STD, 31, 1023, 0.9, 36),
]


def problem(case, c_list):
    kind, m, n, alpha, seed = case
    cfg = synth.Config("small", m, n, kind, min(5, n), 1.0, 2.0, 5.0, alpha, tuple(c_list), seed)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    lm = float(np.max(np.abs(oracle.aty(A, b)))) / alpha
    return cfg, A, b, lm


@pytest.fixture(params=[1, 0], ids=["cluster", "one-cta"])
def small_cl(request):
    return request.param


def use(P, variant):
    P.set_option("small_cluster", variant)
    assert P.info("small_cluster") == variant


def parity(A, b, l1, l2, xg, xc):
    Fg, Fc = oracle.primal_obj(A, b, xg, l1, l2), oracle.primal_obj(A, b, xc, l1, l2)
    return solution_parity(xg, xc, Fg, Fc)


@pytest.mark.parametrize("case", SHAPES, ids=lambda c: f"m{c[1]}_n{c[2]}")
def test_small_matches_oracle_and_graph(case, small_cl):
    cs = (0.5, 0.1, 0.02)  # small c: r ≥ m steps (Eq. (18) branch)
    cfg, A, b, lm = problem(case, cs)
    seen = [0, 0, 0]
    with Problem(A, b) as P:
        assert P.info("small") == 1
        use(P, small_cl)
        for c in cs:
            l1, l2 = c * cfg.alpha * lm, c * (1 - cfg.alpha) * lm
            xc, _, sc, _ = oracle.solve(A, b, l1, l2, sigma0=cfg.sigma0, tol=cfg.tol)
            xs, ss = P.solve(l1, l2, cfg.sigma0, cfg.tol)
            P.set_option("small", 0)
            xg, sg = P.solve(l1, l2, cfg.sigma0, cfg.tol)
            P.set_option("small", 1)
            assert ss["status"] == 0 and sc["status"] == 0, (ss, sc)
            par = parity(A, b, l1, l2, xs, xc)
            assert par["ok"], (c, par, ss, sc)
            assert ss["outer_iters"] == sc["outer_iters"] == sg["outer_iters"]
            assert abs(ss["newton_iters"] - sc["newton_iters"]) <= 1
            assert abs(ss["newton_iters"] - sg["newton_iters"]) <= 1
            # statistics: one Aᵀ pass per Newton step (cold start), the objective of the returned x
            assert ss["aty_passes"] == ss["newton_iters"]
            assert sum(ss["branch_steps"]) == ss["newton_iters"] + ss["jitter_retries"]
            assert ss["active"] == np.count_nonzero(xs)
            assert ss["primal_obj"] == pytest.approx(oracle.primal_obj(A, b, xs, l1, l2), rel=1e-12)
            assert ss["gap"] >= -1e-9 * abs(ss["primal_obj"])
            assert ss["kernel_launches"] < sg["kernel_launches"]
            for k in range(3):
                seen[k] += ss["branch_steps"][k]
    if case[2] >= case[1]:
        assert seen[1] > 0 or seen[2] > 0, seen


def test_small_warm_path_and_pins(small_cl):
    case = SHAPES[0]
    cs = tuple(np.linspace(0.9, 0.1, 10))
    cfg, A, b, lm = problem(case, cs)
    with Problem(A, b) as P:
        use(P, small_cl)
        # x = 0 at λ1 = ‖Aᵀb‖∞ after exactly one Newton step
        g = P.lambda_max_l1
        x, st = P.solve(g, 0.2 * g, 5e-3, 1e-6)
        assert np.all(x == 0) and st["newton_iters"] == 1 and st["outer_iters"] == 1 and st["aty_passes"] == 1
        # warm-started path against the oracle's warm-started path
        x0g = x0c = None
        for c in cs:
            l1, l2 = c * cfg.alpha * lm, c * (1 - cfg.alpha) * lm
            xc, _, sc, _ = oracle.solve(A, b, l1, l2, sigma0=cfg.sigma0, tol=cfg.tol, x0=x0c)
            xs, ss = P.solve(l1, l2, cfg.sigma0, cfg.tol, x0=x0g)
            assert parity(A, b, l1, l2, xs, xc)["ok"], (c, ss, sc)
            assert ss["outer_iters"] == sc["outer_iters"] and abs(ss["newton_iters"] - sc["newton_iters"]) <= 1
            assert ss["aty_passes"] == ss["newton_iters"] + (1 if x0g is not None and np.any(x0g) else 0)
            x0g, x0c = xs, xc
        # warm start at the solution: one outer iteration, no Newton step
        l1, l2 = 0.5 * cfg.alpha * lm, 0.5 * (1 - cfg.alpha) * lm
        xsol, _, _, _ = oracle.solve(A, b, l1, l2, tol=1e-12)
        x, st = P.solve(l1, l2, 5e-3, 1e-6, x0=xsol)
        assert st["outer_iters"] == 1 and st["newton_iters"] == 0 and st["aty_passes"] == 1
        assert np.max(np.abs(x - xsol)) <= 1e-8 * np.max(np.abs(xsol))


def test_small_lasso_innertol_retry_cap(small_cl):
    case = SHAPES[0]
    cfg, A, b, lm = problem(case, (0.3,))
    l1, l2 = 0.3 * cfg.alpha * lm, 0.3 * (1 - cfg.alpha) * lm
    with Problem(A, b) as P:
        use(P, small_cl)
        # Lasso: λ2 = 0, dual objective NaN
        xc, _, _, _ = oracle.solve(A, b, l1, 0.0)
        xs, ss = P.solve(l1, 0.0, 5e-3, 1e-6)
        assert np.isnan(ss["dual_obj"]) and parity(A, b, l1, 0.0, xs, xc)["ok"]
        # adaptive inner tolerance (R37) against the oracle with the same schedule
        P.set_option("inner_tol_mode", 1)
        xc, _, sc, _ = oracle.solve(A, b, l1, l2, inner_tol_mode=1)
        xs, ss = P.solve(l1, l2, 5e-3, 1e-6)
        assert ss["outer_iters"] == sc["outer_iters"] and abs(ss["newton_iters"] - sc["newton_iters"]) <= 1
        assert parity(A, b, l1, l2, xs, xc)["ok"]
        P.set_option("inner_tol_mode", 0)
        # one injected factor failure is retried with the jitter (R36); two are SSNAL_ENUMERIC
        x0, s0 = P.solve(l1, l2, 5e-3, 1e-6)
        P.set_option("test_fail_factor", 1)
        x1, s1 = P.solve(l1, l2, 5e-3, 1e-6)
        assert s1["status"] == 0 and s1["jitter_retries"] == 1
        assert np.max(np.abs(x1 - x0)) <= 1e-8 * np.max(np.abs(x0))
        P.set_option("test_fail_factor", 2)
        _, s2 = P.solve(l1, l2, 5e-3, 1e-6)
        assert s2["status"] == 4  # SSNAL_ENUMERIC
        P.set_option("test_fail_factor", 0)
        # iteration cap: status NOT_CONVERGED with x and stats written
        P.set_option("max_outer", 2)
        xc2, sc2 = P.solve(l1, l2, 5e-3, 1e-6)
        assert sc2["status"] == 1 and sc2["outer_iters"] == 2 and np.any(xc2)
        P.set_option("max_outer", 100)
        x2, s2 = P.solve(l1, l2, 5e-3, 1e-6)
        assert s2["status"] == 0 and np.array_equal(x2, x0)


@pytest.mark.parametrize("m,n,eligible", [(64, 1024, 1), (65, 100, 0), (10, 1025, 0), (2, 1, 1)])
def test_small_eligibility(m, n, eligible):
    """The one-CTA path serves m ≤ 64, n ≤ 1024 (fp64 storage, unsharded, no CG strategy); the option
    small = 0 and the CG strategy turn it off."""
    rng = np.random.default_rng(m * 7 + n)
    A = rng.standard_normal((n, m))
    b = rng.standard_normal(m)
    with Problem(A, b) as P:
        assert P.info("small") == eligible
        if eligible:
            P.set_option("cg_ratio", 2.0)
            assert P.info("small") == 0
            P.set_option("cg_ratio", 0.0)
            P.set_option("small", 0)
            assert P.info("small") == 0
