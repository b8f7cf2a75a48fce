"""Compressed genotype storage: a handle built from packed 2-bit codes + per-column
tables against the oracle run on the decoded fp64 design (bit-identical to synth.design):
K1g (fused Aᵀy over codes), the gathered kernels through the code accessor, whole solves, the
model-selection path, graph ≡ host, validation, and the device generator vs the host one."""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import aty_errors, cuda_ok, dev, empty, host, solution_parity

pytestmark = pytest.mark.gpu

if cuda_ok():
    import torch
    from paper_2006_03970_b200 import Problem, SsnalError


def geno(m, n, seed=4):
    cfg = synth.Config("g", m, n, synth.GENO_STD, 10, 0.1, 0.3, 1.0, 0.5, (0.3,), seed)
    codes, tab = synth.geno_codes(cfg)
    A = synth.decode_geno(codes, tab, m)
    b, _ = synth.response(cfg)
    return cfg, codes, tab, A, b


@pytest.mark.parametrize("m,n", [(800, 5000), (200, 7003), (50, 3000), (33, 1001)])
def test_k1g_parity(m, n):
    """K1g vs the oracle's fused evaluation on the decoded design (R21 tolerances, J bit-exact)."""
    cfg, codes, tab, A, b = geno(m, n, seed=m)
    y = synth.normals(m, 1, m)
    x = np.zeros(n)
    nz = np.arange(0, n, 97)
    x[nz] = synth.normals(m, 2, len(nz))
    sigma, l2 = 0.8, 0.3
    w_ref = oracle.aty(A, y)
    l1 = float(np.quantile(np.abs(x - sigma * w_ref) / sigma, 0.97))
    w_c, J_c, PJ_c, part_c, g_c = oracle.aty_fused(A, b, y, x, sigma, l1, l2)
    with Problem.from_geno(codes, tab, b) as P:
        assert P.info("format") == 1
        dy, dx = dev(y), dev(x)
        w, J, PJ, gg = empty(n), empty(n, torch.int32), empty(n), empty(m)
        r, part = P.aty_fused(dy.data_ptr(), dx.data_ptr(), sigma, l1, l2, w.data_ptr(), J.data_ptr(), PJ.data_ptr(),
                              gg.data_ptr())
        torch.cuda.synchronize()
        e1, e2 = aty_errors(host(w, n), w_c, A, y)
        assert e1 <= 1e-12 and e2 <= 1e-12, (e1, e2)
        assert r == len(J_c) and np.array_equal(host(J, r).astype(np.int64), J_c)
        # P = prox(x − σw) inherits w's error, bounded by R21 relative to ‖a_i‖‖y‖
        scale = sigma * float(np.max(np.sqrt((A * A).sum(axis=1)))) * float(np.linalg.norm(y))
        np.testing.assert_allclose(host(PJ, r), PJ_c, rtol=1e-12, atol=1e-12 * scale)
        np.testing.assert_allclose(part, part_c, rtol=1e-11)
        np.testing.assert_allclose(host(gg, m), g_c, rtol=1e-10, atol=1e-10 * np.abs(g_c).max())
        # λmax of the handle = ‖Aᵀb‖∞ of the decoded design
        assert P.lambda_max_l1 == pytest.approx(float(np.max(np.abs(oracle.aty(A, b)))), rel=1e-12)


@pytest.mark.parametrize("r", [0, 40, 199, 450])
def test_geno_newton_direction(r):
    m, n = 200, 1500
    cfg, codes, tab, A, b = geno(m, n, seed=9)
    J = np.sort(np.argsort(synth.uniforms(9, 7, n))[:r]).astype(np.int64)
    g = synth.normals(9, 8, m)
    kappa = 0.05
    d_cpu, br_cpu = oracle.newton_direction(A, J, g, kappa)
    with Problem.from_geno(codes, tab, b) as P:
        for cg in (0.0, 1e-9):
            P.set_option("cg_ratio", cg)
            dJ, dg, dd = dev(J.astype(np.int32)), dev(g), empty(m)
            gd, br = P.newton_direction(dJ.data_ptr() if r else 0, r, dg.data_ptr(), kappa, dd.data_ptr())
            torch.cuda.synchronize()
            d = host(dd, m)
            if r and cg:
                assert br == 3
            else:
                assert br == br_cpu
            assert np.max(np.abs(d - d_cpu)) <= 1e-8 * np.max(np.abs(d_cpu))


@pytest.mark.parametrize("m,n", [(800, 20_000), (200, 12_000), (50, 4000)])
def test_geno_solve_matches_oracle_and_fp64(m, n):
    cfg, codes, tab, A, b = geno(m, n, seed=m + 1)
    lm = float(np.max(np.abs(oracle.aty(A, b)))) / cfg.alpha
    with Problem.from_geno(codes, tab, b) as G, Problem(A, b) as F:
        for c in (0.5, 0.3):
            l1, l2 = c * cfg.alpha * lm, c * (1 - cfg.alpha) * lm
            xg, sg = G.solve(l1, l2, cfg.sigma0, cfg.tol)
            xf, sf = F.solve(l1, l2, cfg.sigma0, cfg.tol)
            xc, _, sc, _ = oracle.solve(A, b, l1, l2, sigma0=cfg.sigma0, tol=cfg.tol)
            assert sg["status"] == 0 and sc["status"] == 0, (sg, sc)
            Fg = oracle.primal_obj(A, b, xg, l1, l2)
            Fc = oracle.primal_obj(A, b, xc, l1, l2)
            assert solution_parity(xg, xc, Fg, Fc)["ok"], (c, sg, sc)
            assert sg["outer_iters"] == sc["outer_iters"]
            assert abs(sg["newton_iters"] - sc["newton_iters"]) <= 1
            assert sg["primal_obj"] == pytest.approx(Fg, rel=1e-12)
            # same problem as the fp64 handle: same iteration, solutions within rounding
            assert sg["outer_iters"] == sf["outer_iters"]
            assert np.max(np.abs(xg - xf)) <= 1e-8 * np.max(np.abs(xf))


def test_geno_graph_equals_host_and_select():
    m, n = 300, 8000
    cfg, codes, tab, A, b = geno(m, n, seed=17)
    lm = float(np.max(np.abs(oracle.aty(A, b)))) / cfg.alpha
    l1, l2 = 0.3 * cfg.alpha * lm, 0.3 * (1 - cfg.alpha) * lm
    with Problem.from_geno(codes, tab, b) as P:
        P.set_option("graph", 0)
        xh, sh = P.solve(l1, l2)
        P.set_option("graph", 1)
        xg, sg = P.solve(l1, l2)
        assert np.array_equal(xh, xg) and sh["newton_iters"] == sg["newton_iters"]
        crit, xdb = P.model_select(l2, True)
    r, nu, rss, gcv, ebic, xdb_c = oracle.model_select(A, b, xg, l2)
    assert crit["active"] == r
    assert crit["nu"] == pytest.approx(nu, rel=1e-9)
    assert crit["rss"] == pytest.approx(rss, rel=1e-8)
    assert crit["gcv"] == pytest.approx(gcv, rel=1e-8) and crit["ebic"] == pytest.approx(ebic, rel=1e-8, abs=1e-10)
    np.testing.assert_allclose(xdb, xdb_c, rtol=1e-7, atol=1e-9 * np.abs(xdb_c).max())


def test_geno_validation():
    m, n = 40, 200
    cfg, codes, tab, A, b = geno(m, n, seed=21)
    bad = codes.copy()
    bad[5, 0] |= 3  # a code of value 3
    with pytest.raises(SsnalError):
        Problem.from_geno(bad, tab, b)
    t2 = tab.copy()
    t2[7, 1] = np.nan
    if np.any(((codes[7, :] >> 2 * np.arange(4)[:, None]) & 3) == 1):
        with pytest.raises(SsnalError):
            Problem.from_geno(codes, t2, b)
    t3 = tab.copy()
    t3[9, :] = 0.0  # decoded column all zero
    with pytest.raises(SsnalError):
        Problem.from_geno(codes, t3, b)
    with pytest.raises(SsnalError):  # stride not a multiple of 16
        Problem.from_geno(codes[:, :12], tab, b)


@pytest.mark.parametrize("m,n", [(800, 2_000_000)])
def test_geno_device_generator_and_fullsize(m, n):
    """cfg4 at full size in packed form: device generator = host generator on sampled columns; the
    solve converges and satisfies the KKT inclusion on the support and 20 000 sampled columns."""
    cfg = synth.CONFIGS["cfg4"]
    stride = synth.geno_stride(cfg.m)
    st = torch.cuda.current_stream()
    dcodes = torch.empty((cfg.n, stride), dtype=torch.uint8, device="cuda")
    dtab = torch.empty((cfg.n, 3), dtype=torch.float64, device="cuda")
    synth.fill_device_geno(cfg, dcodes.data_ptr(), dtab.data_ptr(), st.cuda_stream)
    b, _ = synth.response(cfg)
    db = torch.from_numpy(b).cuda()
    idx = np.unique(np.minimum((synth.uniforms(3, 31, 64) * cfg.n).astype(np.int64), cfg.n - 1))
    for j in idx[:8]:
        c, t = synth.geno_codes(cfg, int(j), int(j) + 1)
        assert np.array_equal(dcodes[j].cpu().numpy(), c[0]) and np.array_equal(dtab[j].cpu().numpy(), t[0])
    P = Problem.from_geno_device(dcodes.data_ptr(), stride, dtab.data_ptr(), db.data_ptr(), cfg.m, cfg.n,
                                 st.cuda_stream, keep=(dcodes, dtab, db))
    lm = P.lambda_max_l1 / cfg.alpha
    c = cfg.cs[0]
    l1, l2 = c * cfg.alpha * lm, c * (1 - cfg.alpha) * lm
    x, s = P.solve(l1, l2, cfg.sigma0, cfg.tol)
    assert s["status"] == 0 and s["outer_iters"] <= 8
    xt, _ = P.solve(l1, l2, cfg.sigma0, 1e-10, x0=x)
    supp = np.nonzero(xt)[0]
    cols = synth.columns(cfg, supp)
    res = b - cols.T @ xt[supp]
    samp = np.unique(np.concatenate([np.minimum((synth.uniforms(5, 3, 20_000) * cfg.n).astype(np.int64),
                                                cfg.n - 1), supp]))
    C = synth.columns(cfg, samp)
    cval = C @ res - l2 * xt[samp]
    xs = xt[samp]
    v = np.where(xs > 0, np.abs(cval - l1), np.where(xs < 0, np.abs(cval + l1), np.maximum(np.abs(cval) - l1, 0)))
    assert v.max() <= 1e-7 * l1
    P.close()
