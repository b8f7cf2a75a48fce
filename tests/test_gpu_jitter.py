"""The factor retry of S:227 / SURVEY §8(b) (reading R36) on the GPU: the direction hook on
matrices whose Cholesky fails in fp64 (duplicated columns, κ = 1e25) against the oracle's
jittered direction, and whole solves with injected factor failures (option test_fail_factor):
one failure is retried and the solve converges, graph ≡ host bitwise; a failed retry (or
jitter = 0) returns SSNAL_ENUMERIC in both control modes."""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import cuda_ok, dev, empty, host, solution_parity

pytestmark = pytest.mark.gpu

if cuda_ok():
    import torch
    from paper_2006_03970_b200 import Problem, SsnalError


def dup_problem(m, r, seed):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal(m)
    A = np.ascontiguousarray(np.tile(a, (r, 1)))
    b = rng.standard_normal(m)
    g = rng.standard_normal(m)
    return A, b, g


@pytest.mark.parametrize("m,r,br", [(40, 64, 2), (64, 12, 1), (300, 400, 2), (500, 200, 1), (600, 700, 2)])
def test_hook_retry_matches_oracle_jittered(m, r, br):
    """N = min(m, r) covers the three K4 kernels: k_chol_dsm (≤ 160), k_chol_d2 (161–512) and
    k_chol_cluster (> 512)."""
    A, b, g = dup_problem(m, r, seed=m)
    kappa = 1e25
    J = np.arange(r, dtype=np.int32)
    d_c, br_c = oracle.newton_direction(A, J.astype(np.int64), g, kappa, jitter=1e-10)
    assert br_c == br
    with Problem(A, b) as P:
        dJ, dg, dd = dev(J), dev(g), empty(m)
        P.set_option("jitter", 0.0)
        with pytest.raises(SsnalError):
            P.newton_direction(dJ.data_ptr(), r, dg.data_ptr(), kappa, dd.data_ptr())
        P.set_option("jitter", 1e-10)
        gd, b_g = P.newton_direction(dJ.data_ptr(), r, dg.data_ptr(), kappa, dd.data_ptr())
        torch.cuda.synchronize()
        d = host(dd, m)
    assert b_g == br
    # both solve the same jittered system, condition ~ r/jitter: agreement to ~cond·ε
    assert np.linalg.norm(d - d_c) <= 1e-4 * np.linalg.norm(g)
    assert gd < 0


@pytest.mark.parametrize("c", [0.5, 0.1])
def test_solve_with_injected_failure(c):
    cfg = synth.scaled(synth.CONFIGS["cfg2"], n=20_000)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    lm = float(np.max(np.abs(oracle.aty(A, b)))) / cfg.alpha
    l1, l2 = c * cfg.alpha * lm, c * (1 - cfg.alpha) * lm
    xc, _, sc, _ = oracle.solve(A, b, l1, l2, sigma0=cfg.sigma0, tol=cfg.tol)
    with Problem(A, b) as P:
        x0, s0 = P.solve(l1, l2, cfg.sigma0, cfg.tol)
        assert s0["jitter_retries"] == 0
        P.set_option("test_fail_factor", 1)
        out = {}
        for gmode in (0, 1):
            P.set_option("graph", gmode)
            out[gmode] = P.solve(l1, l2, cfg.sigma0, cfg.tol)
        (xh, sh), (xg, sg) = out[0], out[1]
        assert np.array_equal(xh, xg)
        for k in ("status", "jitter_retries", "outer_iters", "newton_iters", "backtracks", "branch_steps",
                  "res_kkt1", "res_kkt3"):
            assert sh[k] == sg[k], (k, sh[k], sg[k])
        assert sg["status"] == 0 and sg["jitter_retries"] == 1
        # the retried step redid one trial pass, nothing else changes the iteration count much
        assert sg["aty_passes"] == s0["aty_passes"] + 1 or abs(sg["newton_iters"] - s0["newton_iters"]) <= 1
        Fg = oracle.primal_obj(A, b, xg, l1, l2)
        Fc = oracle.primal_obj(A, b, xc, l1, l2)
        assert solution_parity(xg, xc, Fg, Fc)["ok"]
        # a failed retry, or no retry allowed: SSNAL_ENUMERIC in both modes
        for inject, jit in ((2, 1e-10), (1, 0.0)):
            P.set_option("test_fail_factor", inject)
            P.set_option("jitter", jit)
            for gmode in (0, 1):
                P.set_option("graph", gmode)
                _, s = P.solve(l1, l2, cfg.sigma0, cfg.tol)
                assert s["status"] == 4, (inject, jit, gmode, s)
                assert s["jitter_retries"] == (1 if jit > 0 else 0)
        P.set_option("test_fail_factor", 0)
        P.set_option("jitter", 1e-10)
        x1, s1 = P.solve(l1, l2, cfg.sigma0, cfg.tol)
        assert np.array_equal(x1, x0)  # the handle recovers: next solve is the plain one
