"""Input generator checks (synth/): determinism, slicing consistency and the
distributional recipe of DESIGN.md ("Input recipe")."""
import numpy as np
import pytest
from scipy import stats

import synth


def test_normals_are_standard_normal():
    x = synth.normals(123, 0, 400_000)
    ks = stats.kstest(x, "norm")
    assert ks.pvalue > 1e-3
    assert abs(x.mean()) < 0.01 and abs(x.std() - 1) < 0.01
    assert np.array_equal(x, synth.normals(123, 0, 400_000))  # deterministic
    assert not np.array_equal(x[:100], synth.normals(124, 0, 100))


def test_uniforms():
    u = synth.uniforms(5, 1, 200_000)
    assert u.min() >= 0 and u.max() < 1
    assert stats.kstest(u, "uniform").pvalue > 1e-3


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
def test_slices_and_columns_agree(name):
    cfg = synth.scaled(synth.CONFIGS[name], n=1200)
    A = synth.design(cfg)
    assert A.shape == (1200, cfg.m)
    # arbitrary windows (crossing AR(1) chunk boundaries at 256, 512, ...)
    for j0, j1 in [(0, 7), (250, 520), (511, 513), (1199, 1200)]:
        assert np.array_equal(synth.design(cfg, j0, j1), A[j0:j1])
    idx = np.array([0, 255, 256, 700, 1199])
    assert np.array_equal(synth.columns(cfg, idx), A[idx])


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4"])
def test_standardisation(name):
    cfg = synth.scaled(synth.CONFIGS[name], n=2000)
    A = synth.design(cfg)
    assert np.max(np.abs(A.mean(axis=1))) < 1e-12
    target = 1.0 if name == "cfg1" else float(cfg.m)
    assert np.allclose((A * A).sum(axis=1), target, rtol=1e-12)


def test_ar1_correlation():
    """cfg2: corr(a_i, a_j) ≈ 0.5^|i−j| (Toeplitz Σ of BASELINE configs[1]; reading R19)."""
    cfg = synth.scaled(synth.CONFIGS["cfg2"], n=3000)
    A = synth.design(cfg) / np.sqrt(cfg.m)
    for lag, rho in [(1, 0.5), (2, 0.25), (3, 0.125), (10, 0.0)]:
        c = np.mean(np.sum(A[:-lag] * A[lag:], axis=1))
        assert abs(c - rho) < 0.02, (lag, c)


def test_genotype_codes_and_linkage():
    """cfg4: each column takes ≤ 3 values (codes 0/1/2 standardised); positive in-block linkage,
    ~no correlation across blocks (reading R18)."""
    cfg = synth.scaled(synth.CONFIGS["cfg4"], n=4000)
    A = synth.design(cfg) / np.sqrt(cfg.m)
    for j in range(0, 4000, 397):
        assert len(np.unique(A[j])) <= 3
    inblock = [np.dot(A[j], A[j + 1]) for j in range(0, 4000, 20)]
    cross = [np.dot(A[j + 19], A[j + 20]) for j in range(0, 3960, 20)]
    assert np.mean(inblock) > 0.2
    assert abs(np.mean(cross)) < 0.02


def test_truth_and_response():
    for name in ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"]:
        cfg = synth.CONFIGS[name]
        idx, val = synth.truth(cfg)
        assert len(idx) == cfg.k and len(np.unique(idx)) == cfg.k
        assert np.all(np.diff(idx) > 0) and idx.min() >= 0 and idx.max() < cfg.n
        assert np.all((np.abs(val) >= cfg.lo) & (np.abs(val) <= cfg.hi))
    cfg = synth.CONFIGS["cfg1"]
    A = synth.design(cfg)
    idx, val = synth.truth(cfg)
    b, sd = synth.response(cfg)
    signal = A[idx].T @ val
    # SNR = var(A x*)/s² (reading R16)
    assert signal.var() / sd ** 2 == pytest.approx(cfg.snr, rel=1e-12)
    assert abs(np.std(b - signal) / sd - 1) < 0.3  # m = 50 noise draws


# ---- compressed genotype storage ----
import pytest  # noqa: E402


@pytest.mark.parametrize("m,n", [(800, 300), (50, 500), (129, 64), (1024, 40), (2, 5000)])
def test_geno_codes_decode_bitwise(m, n):
    """Packed 2-bit codes + per-column tables decode to the fp64 GENO design bit for bit."""
    cfg = synth.scaled(synth.CONFIGS["cfg4"], n=n, m=m)
    codes, tab = synth.geno_codes(cfg)
    assert codes.shape == (n, synth.geno_stride(m)) and synth.geno_stride(m) % 16 == 0
    D = synth.decode_geno(codes, tab, m)
    try:
        A = synth.design(cfg)
    except RuntimeError:  # zero-variance columns (tiny m): compare the non-degenerate columns
        A = None
    if A is not None:
        assert np.array_equal(A, D)
    # every code is 0, 1 or 2; bits beyond row m are zero
    k = np.arange(4 * codes.shape[1])
    g = (codes[:, k // 4] >> (2 * (k % 4))) & 3
    assert g.max() <= 2 and not np.any(g[:, m:])


def test_geno_codes_chunks_consistent():
    cfg = synth.scaled(synth.CONFIGS["cfg4"], n=1000, m=64)
    c, t = synth.geno_codes(cfg)
    c2, t2 = synth.geno_codes(cfg, 300, 700)
    assert np.array_equal(c[300:700], c2) and np.array_equal(t[300:700], t2)
