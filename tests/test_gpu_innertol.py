"""The adaptive inner tolerance (option inner_tol_mode = 1, reading R37) on the GPU: whole
solves against the oracle run with the same schedule (same outer count, Newton count ±1, the
solution parity of BASELINE.json), and graph-mode control ≡ host-mode control bitwise."""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import cuda_ok, solution_parity

pytestmark = pytest.mark.gpu

if cuda_ok():
    from paper_2006_03970_b200 import Problem


@pytest.mark.parametrize("name,n", [("cfg1", None), ("cfg2", 20_000), ("cfg3", 20_000)])
def test_inner_tol_mode_matches_oracle(name, n):
    cfg = synth.CONFIGS[name] if n is None else synth.scaled(synth.CONFIGS[name], n=n)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    lm = float(np.max(np.abs(oracle.aty(A, b)))) / cfg.alpha
    with Problem(A, b) as P:
        P.set_option("inner_tol_mode", 1)
        for c in (0.5, 0.2, 0.1):
            l1, l2 = c * cfg.alpha * lm, c * (1 - cfg.alpha) * lm
            xc, _, sc, _ = oracle.solve(A, b, l1, l2, sigma0=cfg.sigma0, tol=cfg.tol, inner_tol_mode=1)
            out = {}
            P.set_option("small", 0)  # graph ≡ host on the multi-kernel paths
            for g in (0, 1):
                P.set_option("graph", g)
                out[g] = P.solve(l1, l2, cfg.sigma0, cfg.tol)
            P.set_option("small", 1)
            if P.info("small"):  # the one-CTA path (cfg1) with the same schedule
                xs, ss = P.solve(l1, l2, cfg.sigma0, cfg.tol)
                assert ss["status"] == 0 and ss["outer_iters"] == sc["outer_iters"]
                assert abs(ss["newton_iters"] - sc["newton_iters"]) <= 1
                assert solution_parity(xs, xc, oracle.primal_obj(A, b, xs, l1, l2),
                                       oracle.primal_obj(A, b, xc, l1, l2))["ok"], (c, ss, sc)
            (xh, sh), (xg, sg) = out[0], out[1]
            assert np.array_equal(xh, xg)
            for k in ("outer_iters", "newton_iters", "backtracks", "branch_steps", "res_kkt1", "res_kkt3"):
                assert sh[k] == sg[k], (k, sh[k], sg[k])
            assert sg["status"] == 0 and sc["status"] == 0
            assert sg["outer_iters"] == sc["outer_iters"]
            assert abs(sg["newton_iters"] - sc["newton_iters"]) <= 1
            Fg = oracle.primal_obj(A, b, xg, l1, l2)
            Fc = oracle.primal_obj(A, b, xc, l1, l2)
            assert solution_parity(xg, xc, Fg, Fc)["ok"], (c, sg, sc)
