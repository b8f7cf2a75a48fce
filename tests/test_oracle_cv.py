"""Pins for the oracle's k-fold cross-validation along the λ path (Section 3.3, P:393-412;
SURVEY §8(f1); reading R35: interleaved folds r ≡ f (mod k), the full-data λ grid, CV error =
Σ_folds ‖b_test − A_test x_fold‖² / m).

Independent of the oracle's own solver: scikit-learn's coordinate-descent ElasticNet on the same
folds (its objective ×m_train is Eq. (1) with λ1 = m_train·α·ρ, λ2 = m_train·α·(1−ρ)), and the
closed form above every fold's λmax (x = 0 ⇒ CV = ‖b‖²/m exactly)."""
import numpy as np
import pytest

import oracle
import synth


def small(seed=3, m=40, n=120):
    cfg = synth.Config("cv", m, n, synth.IID_STD, 6, 1.0, 2.0, 5.0, 0.7, (0.5,), seed)
    return cfg, synth.design(cfg), synth.response(cfg)[0]


def test_folds_partition_rows():
    for m, k in [(40, 5), (41, 5), (10, 10), (7, 3)]:
        f = oracle.cv_folds(m, k)
        allr = np.sort(np.concatenate(f))
        assert np.array_equal(allr, np.arange(m)) and len(f) == k


def test_cv_above_every_fold_lambda_max_is_norm_b():
    cfg, A, b = small()
    m = cfg.m
    lm = float(np.max(np.abs(oracle.aty(A, b)))) / cfg.alpha
    worst = 0.0
    for test in oracle.cv_folds(m, 5):
        train = np.setdiff1d(np.arange(m), test)
        worst = max(worst, float(np.max(np.abs(oracle.aty(np.ascontiguousarray(A[:, train]), b[train])))))
    c = 1.01 * worst / (cfg.alpha * lm)
    err, _ = oracle.cv_path(A, b, cfg.alpha, [c], k=5)
    assert err[0] == pytest.approx(float(b @ b) / m, rel=1e-15)


def test_cv_matches_sklearn_elasticnet():
    sk = pytest.importorskip("sklearn.linear_model")
    cfg, A, b = small(seed=5, m=36, n=90)
    m = cfg.m
    cs = [0.6, 0.3, 0.15]
    err, best = oracle.cv_path(A, b, cfg.alpha, cs, k=4, tol=1e-10)
    lm = float(np.max(np.abs(oracle.aty(A, b)))) / cfg.alpha
    ref = np.zeros(len(cs))
    for test in oracle.cv_folds(m, 4):
        train = np.setdiff1d(np.arange(m), test)
        X = A[:, train].T  # m_train × n
        for i, c in enumerate(cs):
            l1, l2 = c * cfg.alpha * lm, c * (1 - cfg.alpha) * lm
            a = (l1 + l2) / len(train)
            mdl = sk.ElasticNet(alpha=a, l1_ratio=l1 / (l1 + l2), fit_intercept=False, tol=1e-14, max_iter=1_000_000)
            mdl.fit(X, b[train])
            r = A[:, test].T @ mdl.coef_ - b[test]
            ref[i] += r @ r
    ref /= m
    np.testing.assert_allclose(err, ref, rtol=1e-7)
    assert best == int(np.argmin(ref))
