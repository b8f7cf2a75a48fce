"""K4 variants (Eq. (18)/(19) factor and solves): the DSMEM-resident cluster
Cholesky (k_chol_dsm, N ≤ 96) and the split-ownership DSMEM Cholesky (k_chol_d2, 96 < N ≤ 512)
against the L2-tiled cluster Cholesky (k_chol_cluster) and the oracle, through the
Newton-direction hook, across tile edges and the switch points; and whole solves with each
variant, graph-mode control ≡ host-mode control."""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import cuda_ok, dev, empty, host

pytestmark = pytest.mark.gpu

if cuda_ok():
    import torch
    from paper_2006_03970_b200 import Problem


def direction(P, J, g, kappa):
    m = len(g)
    dJ, dg, dd = dev(J.astype(np.int32)), dev(g), empty(m)
    gd, br = P.newton_direction(dJ.data_ptr() if len(J) else 0, len(J), dg.data_ptr(), kappa, dd.data_ptr())
    torch.cuda.synchronize()
    return host(dd, m), gd, br


@pytest.mark.parametrize("m,r", [(500, 1), (500, 31), (500, 32), (500, 33), (500, 96), (500, 97), (500, 100), (500, 160), (500, 161),
                                 (500, 300), (160, 159), (160, 400), (161, 400), (40, 7), (64, 1000),
                                 (500, 192), (500, 255), (500, 256), (500, 257), (500, 435), (500, 499),
                                 (500, 500), (500, 700), (511, 900), (512, 1000), (513, 1000), (400, 2000)])
def test_dsm_vs_cluster_vs_oracle(m, r):
    n = max(2 * r, 1500)
    cfg = synth.Config("k4", m, n, synth.IID_STD, 5, 1.0, 2.0, 5.0, 0.7, (0.5,), m + r)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    J = np.sort(np.argsort(synth.uniforms(m + r, 7, n))[:r]).astype(np.int64)
    g = synth.normals(m + r, 8, m)
    kappa = 0.02
    d_c, br_c = oracle.newton_direction(A, J, g, kappa)
    with Problem(A, b) as P:
        out = {}
        for v, v2 in ((1, 1), (1, 0), (0, 0)):
            P.set_option("chol_dsm", v)
            P.set_option("chol_d2", v2)
            out[v, v2] = direction(P, J, g, kappa)
    (d0, gd0, b0) = out[0, 0]
    scale = np.max(np.abs(d_c))
    for key in ((1, 1), (1, 0)):
        (d1, gd1, b1) = out[key]
        assert b1 == b0 == br_c
        assert np.max(np.abs(d1 - d0)) <= 1e-12 * scale, key
        assert np.max(np.abs(d1 - d_c)) <= 1e-10 * scale, key
        assert gd1 == pytest.approx(gd0, rel=1e-12)


@pytest.mark.parametrize("m,n", [(150, 4000), (300, 8000), (500, 20000)])
def test_solves_with_both_variants(m, n):
    """m = 150: every factor on the DSMEM kernel; m = 300 / 500: k_chol_dsm and k_chol_d2, switching
    on N inside the graph.  Same iteration as the L2-tiled variant up to rounding; graph ≡ host
    bitwise."""
    cfg = synth.Config("k4s", m, n, synth.AR1_STD, 10, 1.0, 2.0, 5.0, 0.7, (0.5,), 11)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    lm = float(np.max(np.abs(oracle.aty(A, b)))) / cfg.alpha
    with Problem(A, b) as P:
        for c in (0.3, 0.05):
            l1, l2 = c * cfg.alpha * lm, c * (1 - cfg.alpha) * lm
            res = {}
            for dsm in (1, 0):
                P.set_option("chol_dsm", dsm)
                for gm in (0, 1):
                    P.set_option("graph", gm)
                    res[dsm, gm] = P.solve(l1, l2, cfg.sigma0, cfg.tol)
            for dsm in (1, 0):
                (xh, sh), (xg, sg) = res[dsm, 0], res[dsm, 1]
                assert np.array_equal(xh, xg), dsm
                assert sh["newton_iters"] == sg["newton_iters"] and sh["branch_steps"] == sg["branch_steps"]
            x1, s1 = res[1, 1]
            x0, s0 = res[0, 1]
            assert s1["status"] == 0 and s0["status"] == 0
            assert s1["outer_iters"] == s0["outer_iters"]
            assert np.max(np.abs(x1 - x0)) <= 1e-8 * np.max(np.abs(x0))
