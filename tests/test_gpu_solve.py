"""End-to-end GPU solve parity with the CPU oracle (BASELINE north-star tolerances), plus the
oracle-free pins that hold at any size (x = 0 above λmax, warm start at the solution,
near-λmax single active coefficient, KKT inclusion on sampled columns)."""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import compare_to_oracle, cuda_ok, solution_parity

pytestmark = pytest.mark.gpu

if cuda_ok():
    from paper_2006_03970_b200 import Problem


def lambdas(cfg, lmax_l1, c):
    """λmax = ‖Aᵀb‖∞/α, λ1 = c α λmax, λ2 = c (1−α) λmax."""
    lmax = lmax_l1 / cfg.alpha
    return c * cfg.alpha * lmax, c * (1 - cfg.alpha) * lmax


def run_pair(A, b, l1, l2, sigma0=5e-3, tol=1e-6, x0=None, P=None):
    xc, yc, stc, _ = oracle.solve(A, b, l1, l2, sigma0=sigma0, tol=tol, x0=x0)
    own = P is None
    if own:
        P = Problem(A, b)
    xg, stg = P.solve(l1, l2, sigma0, tol, x0=x0)
    if own:
        P.close()
    return xc, stc, xg, stg


def check_parity(xc, stc, xg, stg, A, b, l1, l2, label=""):
    assert stg["status"] == 0, (label, stg)
    assert stc["status"] == 0, (label, stc)
    Fg = oracle.primal_obj(A, b, xg, l1, l2)
    Fc = oracle.primal_obj(A, b, xc, l1, l2)
    par = solution_parity(xg, xc, Fg, Fc)
    assert par["ok"], (label, par, stg, stc)
    # the GPU's own objective report agrees with the oracle's evaluation of its x
    assert stg["primal_obj"] == pytest.approx(Fg, rel=1e-12)
    assert stg["gap"] >= -1e-9 * abs(Fg)
    return par


@pytest.mark.parametrize("name,n", [("cfg1", None), ("cfg3", 20_000), ("cfg4", 20_000), ("cfg5", 30_000)])
def test_solve_matches_oracle(name, n):
    cfg = synth.CONFIGS[name] if n is None else synth.scaled(synth.CONFIGS[name], n=n)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    lm = float(np.max(np.abs(oracle.aty(A, b))))
    with Problem(A, b) as P:
        for c in cfg.cs:
            l1, l2 = lambdas(cfg, lm, c)
            # identical iteration (same readings): equal outer and Newton counts, else the ±1 rerun rule;
            # objective, x, sign pattern, dual objective and gap against the oracle
            compare_to_oracle(A, b, l1, l2, lambda s0, tol, x0: P.solve(l1, l2, s0, tol, x0=x0),
                              label=f"{name} c={c}")


def test_cfg2_path_full_size():
    """BASELINE configs[1]: warm-started path over c = 0.9 … 0.1 at full size (m=500, n=1e5), σ carried
    from point to point (reading R38): point by point against the oracle from the same start
    (x0 = the oracle's previous point, σ0 = its sigma_final)."""
    cfg = synth.CONFIGS["cfg2"]
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    lm = float(np.max(np.abs(oracle.aty(A, b))))
    x_prev, sig = None, cfg.sigma0
    with Problem(A, b) as P:
        assert P.lambda_max_l1 == pytest.approx(lm, rel=1e-13)
        for c in cfg.cs:
            l1, l2 = lambdas(cfg, lm, c)
            _, _, stc, _ = compare_to_oracle(A, b, l1, l2, lambda s0, tol, x0: P.solve(l1, l2, s0, tol, x0=x0),
                                             sigma0=sig, x0=x_prev, label=f"path c={c}")
            x_prev, _, st, _ = oracle.solve(A, b, l1, l2, sigma0=sig, tol=cfg.tol, x0=x_prev)
            sig = st["sigma_final"]


def test_zero_above_lambda_max():
    """λ1 ≥ ‖Aᵀb‖∞ ⇒ x = 0 after exactly one Newton step."""
    cfg = synth.scaled(synth.CONFIGS["cfg3"], n=50_000)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    with Problem(A, b) as P:
        g = P.lambda_max_l1  # the GPU's own ‖Aᵀb‖∞: bitwise consistent with its Aᵀ(−b)
        for l1 in (g, 1.5 * g):
            x, st = P.solve(l1, 0.2 * g, 5e-3, 1e-6)
            assert np.all(x == 0) and st["status"] == 0
            assert st["newton_iters"] == 1 and st["outer_iters"] == 1 and st["aty_passes"] == 1


def test_warm_start_at_solution():
    cfg = synth.scaled(synth.CONFIGS["cfg5"], n=40_000)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    lm = float(np.max(np.abs(oracle.aty(A, b))))
    l1, l2 = lambdas(cfg, lm, 0.5)
    xs, _, _, _ = oracle.solve(A, b, l1, l2, tol=1e-12)
    with Problem(A, b) as P:
        x, st = P.solve(l1, l2, 5e-3, 1e-6, x0=xs)
        assert st["outer_iters"] == 1 and st["newton_iters"] == 0 and st["aty_passes"] == 1
        assert np.max(np.abs(x - xs)) <= 1e-8 * np.max(np.abs(xs))


def test_near_lambda_max_single_active():
    cfg = synth.scaled(synth.CONFIGS["cfg3"], n=30_000)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    c = A @ b
    j = int(np.argmax(np.abs(c)))
    g = abs(c[j])
    l1, l2 = g * (1 - 1e-3), 0.2 * g
    xj = np.sign(c[j]) * (g - l1) / (A[j] @ A[j] + l2)
    assert np.max(np.abs(np.delete(A @ (b - A[j] * xj), j))) <= l1
    with Problem(A, b) as P:
        x, st = P.solve(l1, l2, 5e-3, 1e-10)
    # error on the natural coefficient scale g/(‖a‖² + λ2), as in the oracle pin
    assert np.count_nonzero(x) == 1 and abs(x[j] - xj) <= 1e-9 * g / (A[j] @ A[j] + l2)


def test_lasso_lambda2_zero():
    """λ2 = 0 is accepted (Lasso); dual objective reported as NaN."""
    cfg = synth.scaled(synth.CONFIGS["cfg1"], n=400)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    lm = float(np.max(np.abs(oracle.aty(A, b))))
    xc, _, stc, _ = oracle.solve(A, b, 0.3 * lm, 0.0)
    with Problem(A, b) as P:
        xg, stg = P.solve(0.3 * lm, 0.0, 5e-3, 1e-6)
    assert np.isnan(stg["dual_obj"])
    Fg, Fc = oracle.primal_obj(A, b, xg, 0.3 * lm, 0.0), oracle.primal_obj(A, b, xc, 0.3 * lm, 0.0)
    assert abs(Fg - Fc) <= 1e-9 * abs(Fc)


def test_invalid_arguments():
    from paper_2006_03970_b200 import SsnalError

    cfg = synth.scaled(synth.CONFIGS["cfg1"], n=100)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    with Problem(A, b) as P:
        for args in [(-1.0, 1.0, 5e-3, 1e-6), (1.0, -1.0, 5e-3, 1e-6), (0.0, 0.0, 5e-3, 1e-6),
                     (1.0, 1.0, 0.0, 1e-6), (1.0, 1.0, 5e-3, 0.0)]:
            with pytest.raises(SsnalError):
                P.solve(*args)
        with pytest.raises(SsnalError):
            P.set_option("no_such_option", 1)
        for key, bad in (("carry_sigma", 2), ("small_cluster", 3), ("cluster_size", 3), ("cluster_size", 32)):
            with pytest.raises(SsnalError):
                P.set_option(key, bad)
        # cluster_size 0 = auto (the largest schedulable power of two); an explicit schedulable size is kept
        P.set_option("cluster_size", 0)
        auto = P.info("cluster_size")
        assert auto in (1, 2, 4, 8, 16)
        P.set_option("cluster_size", 8)
        assert P.info("cluster_size") == 8
        P.set_option("carry_sigma", 0)
        assert P.info("carry_sigma") == 0


EDGE = [  # (kind, m, n, c, alpha, seed): tiny / odd / largest-m shapes; small c pushes r ≥ m (Eq. (18) branch)
    (synth.IID_STD, 2, 1, 0.5, 0.5, 61),
    (synth.IID_STD, 3, 7, 0.3, 0.7, 62),
    (synth.IID_STD, 33, 100, 0.2, 0.5, 63),
    (synth.IID_UNIT_L2, 129, 5000, 0.1, 0.5, 64),
    (synth.IID_STD, 1024, 2500, 0.1, 0.3, 65),
    (synth.GENO_STD, 200, 3000, 0.05, 0.5, 66),  # genotype columns need enough rows to vary
]


@pytest.mark.parametrize("case", EDGE, ids=lambda c: f"m{c[1]}_n{c[2]}_c{c[3]}")
def test_solve_edge_shapes(case):
    kind, m, n, c, alpha, seed = case
    cfg = synth.Config("edge", m, n, kind, min(5, n), 1.0, 2.0, 5.0, alpha, (c,), seed)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    lm = float(np.max(np.abs(oracle.aty(A, b))))
    l1, l2 = lambdas(cfg, lm, c)
    with Problem(A, b) as P:
        compare_to_oracle(A, b, l1, l2, lambda s0, tol, x0: P.solve(l1, l2, s0, tol, x0=x0), label=f"edge {case}")


@pytest.mark.parametrize("name,n", [("cfg1", None), ("cfg3", 20_000)])
def test_certify_primal_violation(name, n):
    """Option certify: stats.primal_viol = max_i v_i over all n columns (one extra Aᵀ pass), against the
    oracle's definition of the KKT-inclusion violation at the GPU's own x; NaN without the option."""
    cfg = synth.CONFIGS[name] if n is None else synth.scaled(synth.CONFIGS[name], n=n)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    lm = float(np.max(np.abs(oracle.aty(A, b))))
    l1, l2 = lambdas(cfg, lm, cfg.cs[0])
    with Problem(A, b) as P:
        x, st = P.solve(l1, l2, cfg.sigma0, cfg.tol)
        assert np.isnan(st["primal_viol"])
        P.set_option("certify", 1)
        for tol in (cfg.tol, 1e-10):
            x, st = P.solve(l1, l2, cfg.sigma0, tol)
            ref = oracle.kkt_violation(A, b, x, l1, l2)
            assert st["primal_viol"] == pytest.approx(ref, rel=1e-6, abs=1e-12 * l1)
        assert st["primal_viol"] <= 1e-7 * l1


def test_two_live_handles_with_different_k1_rings():
    """Two handles in the same K1 register bucket (m = 300 and m = 500 → MR = 16) but with different ring
    sizes, alive at once: the second create must not lower the first one's dynamic shared-memory cap."""
    cfgs = [synth.scaled(synth.CONFIGS["cfg3"], n=4000, m=500), synth.scaled(synth.CONFIGS["cfg3"], n=4000, m=300)]
    data = [(synth.design(c), synth.response(c)[0]) for c in cfgs]
    with Problem(*data[0]) as P0, Problem(*data[1]) as P1:
        for P, (A, b), cfg in ((P0, data[0], cfgs[0]), (P1, data[1], cfgs[1]), (P0, data[0], cfgs[0])):
            l1, l2 = lambdas(cfg, P.lambda_max_l1, 0.3)
            compare_to_oracle(A, b, l1, l2, lambda s0, tol, x0: P.solve(l1, l2, s0, tol, x0=x0), label="two handles")
