"""Run-to-run determinism as a race check for the cluster and one-CTA kernels (compute-sanitizer is not
available on this pool): every reduction on the GPU path has a fixed order, so repeated launches on the
same inputs must be bitwise identical.  Covers k_chol_d2 (every N class through the Newton-direction
hook, repeated 20 times) and k_small_solve (repeated whole solves)."""
import numpy as np
import pytest

import synth
from gpu_util import cuda_ok, dev, empty, host

pytestmark = pytest.mark.gpu

if cuda_ok():
    import torch
    from paper_2006_03970_b200 import Problem


@pytest.mark.parametrize("m,r", [(500, 161), (500, 200), (500, 320), (500, 435), (500, 511), (512, 600), (300, 900)])
def test_k4_d2_bitwise_repeatable(m, r):
    n = max(2 * r, 2000)
    cfg = synth.Config("det", m, n, synth.IID_STD, 5, 1.0, 2.0, 5.0, 0.7, (0.5,), m + 3 * r)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    J = np.sort(np.argsort(synth.uniforms(r, 7, n))[:r]).astype(np.int32)
    g = synth.normals(r, 8, m)
    with Problem(A, b) as P:
        assert P.info("chol_d2") == 1
        dJ, dg, dd = dev(J), dev(g), empty(m)
        ref = None
        for _ in range(20):
            gd, br = P.newton_direction(dJ.data_ptr(), r, dg.data_ptr(), 0.05, dd.data_ptr())
            torch.cuda.synchronize()
            d = host(dd, m).copy()
            if ref is None:
                ref = (d, gd, br)
            else:
                assert np.array_equal(d, ref[0]) and gd == ref[1] and br == ref[2]


def test_small_solve_bitwise_repeatable():
    cfg = synth.CONFIGS["cfg1"]
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    with Problem(A, b) as P:
        assert P.info("small") == 1
        lm = P.lambda_max_l1 / cfg.alpha
        for c in (0.5, 0.05):
            l1, l2 = c * cfg.alpha * lm, c * (1 - cfg.alpha) * lm
            x0, s0 = P.solve(l1, l2, cfg.sigma0, cfg.tol)
            for _ in range(10):
                x, s = P.solve(l1, l2, cfg.sigma0, cfg.tol)
                assert np.array_equal(x, x0)
                assert s["newton_iters"] == s0["newton_iters"] and s["psi_evals"] == s0["psi_evals"]
