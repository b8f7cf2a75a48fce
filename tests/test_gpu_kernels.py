"""GPU kernel parity (call through the C-ABI): K1 fused pass, K1e epilogue, K2–K4 Newton
direction, each against the CPU oracle on the same seeded inputs (synth/)."""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import aty_errors, cuda_ok, dev, empty, host, separated_threshold

pytestmark = pytest.mark.gpu

if cuda_ok():
    import torch
    from paper_2006_03970_b200 import Problem


def _problem_inputs(kind, m, n, seed):
    cfg = synth.Config("t", m, n, kind, min(5, n), 1.0, 2.0, 5.0, 0.7, (0.5,), seed)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    return cfg, A, b


K1_CASES = [
    # (kind, m, n, seed, r_target)   — several tiles, ragged tails, odd m, tiny n
    (synth.IID_UNIT_L2, 50, 1000, 1, 17),
    (synth.AR1_STD, 500, 3001, 2, 40),
    (synth.IID_STD, 51, 777, 3, 9),
    (synth.GENO_STD, 800, 2049, 4, 100),
    (synth.IID_STD, 2, 5, 5, 2),
    (synth.IID_STD, 3, 1, 6, 1),
    (synth.IID_STD, 1024, 300, 7, 30),
    (synth.IID_STD, 33, 4099, 8, 0),
    (synth.IID_STD, 129, 1500, 9, 1500),
    # many tiles per CTA (ring slots reused by different warps): n ≫ 148 · C · stages
    (synth.IID_STD, 500, 200_003, 10, 300),
    (synth.IID_STD, 64, 300_001, 12, 3000),
    (synth.GENO_STD, 800, 60_001, 13, 500),
]


@pytest.mark.parametrize("case", K1_CASES, ids=lambda c: f"m{c[1]}_n{c[2]}_r{c[4]}")
def test_k1_fused_parity(case):
    kind, m, n, seed, r_target = case
    cfg, A, b = _problem_inputs(kind, m, n, seed)
    y = synth.normals(seed, 1, m)
    x = np.zeros(n)
    nzi = np.unique((synth.uniforms(seed, 2, min(10, n)) * n).astype(np.int64))
    x[nzi] = synth.normals(seed, 3, len(nzi))
    sigma, l2 = 0.7, 0.3
    w_ref = oracle.aty(A, y)
    t = x - sigma * w_ref
    l1 = separated_threshold(t, r_target) / sigma
    w_cpu, J_cpu, PJ_cpu, part_cpu, g_cpu = oracle.aty_fused(A, b, y, x, sigma, l1, l2)
    assert len(J_cpu) == r_target
    with Problem(A, b) as P:
        dy, dx = dev(y), dev(x)
        w, J, PJ, g = empty(n), empty(n, torch.int32), empty(n), empty(m)
        r, part = P.aty_fused(dy.data_ptr(), dx.data_ptr(), sigma, l1, l2, w.data_ptr(), J.data_ptr(),
                              PJ.data_ptr(), g.data_ptr())
        torch.cuda.synchronize()
        e1, e2 = aty_errors(host(w, n), w_cpu, A, y)
        assert e1 <= 1e-12 and e2 <= 1e-12, (e1, e2)
        assert r == r_target
        assert np.array_equal(host(J, r).astype(np.int64), J_cpu)  # bit-exact index work
        np.testing.assert_allclose(host(PJ, r), PJ_cpu, rtol=1e-11, atol=1e-13 * max(1, np.abs(PJ_cpu).max(initial=0)))
        for q in range(4):
            assert part[q] == pytest.approx(part_cpu[q], rel=1e-10, abs=1e-12 * (1 + abs(part_cpu[q])))
        scale = np.linalg.norm(y) + np.linalg.norm(b) + float(np.sum(np.abs(PJ_cpu) * np.sqrt((A[J_cpu] ** 2).sum(1))))
        assert np.max(np.abs(host(g, m) - g_cpu)) <= 1e-12 * scale
        # λmax = ‖Aᵀb‖∞ from the create-time pass
        lm = float(np.max(np.abs(oracle.aty(A, b))))
        assert P.lambda_max_l1 == pytest.approx(lm, rel=1e-13)


@pytest.mark.parametrize("with_w1", [False, True])
def test_k1e_epilogue_parity(with_w1):
    m, n, seed = 64, 5003, 11
    cfg, A, b = _problem_inputs(synth.IID_STD, m, n, seed)
    w0 = synth.normals(seed, 4, n) * 3
    w1 = synth.normals(seed, 5, n) * 3
    x = np.zeros(n)
    x[::97] = synth.normals(seed, 6, len(x[::97]))
    s = 0.25
    weff = w0 + s * (w1 - w0) if with_w1 else w0  # same IEEE op order as the kernel (no FMA)
    sigma, l2 = 1.3, 0.2
    t = x - sigma * weff
    l1 = separated_threshold(t, 70) / sigma
    J_cpu = oracle.active_set(t, sigma, l1)
    P_all = oracle.prox(t, sigma, l1, l2)
    with Problem(A, b) as P:
        d0, d1, dxx = dev(w0), dev(w1), dev(x)
        wo, J, PJ = empty(n), empty(n, torch.int32), empty(n)
        r, part = P.epilogue(d0.data_ptr(), d1.data_ptr() if with_w1 else 0, s, dxx.data_ptr(), sigma, l1, l2,
                             wo.data_ptr(), J.data_ptr(), PJ.data_ptr())
        torch.cuda.synchronize()
        assert np.array_equal(host(wo, n), weff)
        assert r == len(J_cpu) == 70
        assert np.array_equal(host(J, r).astype(np.int64), J_cpu)
        np.testing.assert_array_equal(host(PJ, r), P_all[J_cpu])
        dx_ = x - P_all
        z = dx_ / sigma - weff
        e = np.maximum(np.abs(weff) - l1, 0)
        ref = [P_all @ P_all, dx_ @ dx_, z @ z, e @ e]
        for q in range(4):
            assert part[q] == pytest.approx(ref[q], rel=1e-12)


@pytest.mark.parametrize("r", [0, 1, 31, 32, 33, 99, 100, 101, 250])
def test_newton_direction_parity(r):
    """K2–K4 vs the oracle's Eq. (18)/(19) for r around the tile edges and the r = m switch (m = 100)."""
    m, n, seed = 100, 400, 21
    cfg, A, b = _problem_inputs(synth.IID_STD, m, n, seed)
    J = np.sort((np.argsort(synth.uniforms(seed, 7, n))[:r]).astype(np.int64))
    g = synth.normals(seed, 8, m) * 5
    kappa = 0.37
    d_cpu, br_cpu = oracle.newton_direction(A, J, g, kappa)
    with Problem(A, b) as P:
        dJ, dg, dd = dev(J.astype(np.int32)), dev(g), empty(m)
        gd, br = P.newton_direction(dJ.data_ptr() if r else 0, r, dg.data_ptr(), kappa, dd.data_ptr())
        torch.cuda.synchronize()
        assert br == br_cpu
        d = host(dd, m)
        assert np.max(np.abs(d - d_cpu)) <= 1e-10 * np.max(np.abs(d_cpu))
        assert gd == pytest.approx(g @ d_cpu, rel=1e-10)
        assert gd < 0


@pytest.mark.parametrize("m", [50, 500, 800])
def test_newton_direction_large_r(m):
    """m × m branch at realistic sizes (r ≥ m, split-K Gram, cluster Cholesky)."""
    n, seed = 3 * m + 7, 31
    cfg, A, b = _problem_inputs(synth.IID_STD, m, n, seed)
    r = 2 * m + 3
    J = np.sort((np.argsort(synth.uniforms(seed, 7, n))[:r]).astype(np.int64))
    g = synth.normals(seed, 8, m)
    kappa = 2e-3
    d_cpu, br_cpu = oracle.newton_direction(A, J, g, kappa)
    with Problem(A, b) as P:
        dJ, dg, dd = dev(J.astype(np.int32)), dev(g), empty(m)
        gd, br = P.newton_direction(dJ.data_ptr(), r, dg.data_ptr(), kappa, dd.data_ptr())
        torch.cuda.synchronize()
        assert br == br_cpu == 2
        assert np.max(np.abs(host(dd, m) - d_cpu)) <= 1e-10 * np.max(np.abs(d_cpu))
    # SMW branch just below m
    r = m - 1
    J = J[:r]
    d_cpu, br_cpu = oracle.newton_direction(A, J, g, kappa)
    with Problem(A, b) as P:
        dJ, dg, dd = dev(J.astype(np.int32)), dev(g), empty(m)
        gd, br = P.newton_direction(dJ.data_ptr(), r, dg.data_ptr(), kappa, dd.data_ptr())
        torch.cuda.synchronize()
        assert br == br_cpu == 1
        assert np.max(np.abs(host(dd, m) - d_cpu)) <= 1e-9 * np.max(np.abs(d_cpu))


def test_create_device_and_validation():
    m, n = 40, 300
    cfg, A, b = _problem_inputs(synth.IID_STD, m, n, 41)
    dA, db = dev(A), dev(b)
    P = Problem.from_device(dA.data_ptr(), db.data_ptr(), m, n, torch.cuda.current_stream().cuda_stream,
                            keep=(dA, db))
    assert P.lambda_max_l1 == pytest.approx(float(np.max(np.abs(A @ b))), rel=1e-13)
    P.close()
    from paper_2006_03970_b200 import SsnalError

    A2 = A.copy()
    A2[7] = 0.0
    with pytest.raises(SsnalError):
        Problem(A2, b)
    A3 = A.copy()
    A3[3, 2] = np.nan
    with pytest.raises(SsnalError):
        Problem(A3, b)
    with pytest.raises(SsnalError):
        Problem(np.zeros((5, 1)), np.zeros(1))  # m < 2
