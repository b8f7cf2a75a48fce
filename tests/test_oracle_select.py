"""Pins for the oracle's model-selection pieces (Section 3.3).

ν (degrees of freedom) against the singular-value form Σ σ_i²/(σ_i² + λ2) (a different
computation of the same trace), its limits (λ2 = 0 → r; orthonormal columns → r/(1+λ2)); the
de-biased fit against numpy least squares; Eq. (21) at special values."""
import numpy as np
import pytest

import oracle


def _A(seed, m=20, n=40):
    rng = np.random.default_rng(seed)
    return rng.normal(size=(n, m)), rng.normal(size=m)


@pytest.mark.parametrize("seed", range(5))
@pytest.mark.parametrize("l2", [0.0, 0.3, 7.0])
def test_dof_matches_svd(seed, l2):
    A, _ = _A(seed)
    J = np.array([1, 4, 5, 9, 17, 30])
    s = np.linalg.svd(A[J].T, compute_uv=False)
    ref = float(np.sum(s ** 2 / (s ** 2 + l2)))
    assert oracle.dof(A, J, l2) == pytest.approx(ref, rel=1e-12)


def test_dof_limits():
    A, _ = _A(1)
    J = np.arange(8)
    assert oracle.dof(A, J, 0.0) == pytest.approx(8.0, rel=1e-12)   # λ2 = 0: ν = r (full rank)
    assert oracle.dof(A, np.array([], dtype=np.int64), 2.0) == 0.0
    Q, _ = np.linalg.qr(np.random.default_rng(2).normal(size=(30, 6)))
    Ao = np.ascontiguousarray(Q.T)
    assert oracle.dof(Ao, np.arange(6), 0.5) == pytest.approx(6 / 1.5, rel=1e-12)  # orthonormal: r/(1+λ2)


@pytest.mark.parametrize("seed", range(4))
def test_ols_matches_lstsq(seed):
    A, b = _A(seed)
    J = np.array([0, 3, 7, 8, 21])
    v, rss, ok = oracle.ols(A, b, J)
    ref, res, *_ = np.linalg.lstsq(A[J].T, b, rcond=None)
    assert ok
    np.testing.assert_allclose(v, ref, rtol=1e-10, atol=1e-12)
    assert rss == pytest.approx(float(np.sum((b - A[J].T @ ref) ** 2)), rel=1e-10)


def test_ols_empty_and_singular():
    A, b = _A(3)
    v, rss, ok = oracle.ols(A, b, np.array([], dtype=np.int64))
    assert ok and rss == pytest.approx(float(b @ b), rel=1e-14)
    A2 = A.copy()  # duplicated column with ‖a‖² = 25: the Cholesky pivot is exactly 0
    A2[2] = 0.0
    A2[2, :2] = [3.0, 4.0]
    A2[5] = A2[2]
    _, _, ok = oracle.ols(A2, b, np.array([2, 5]))
    assert not ok


def test_criteria_special_values():
    # ν = 0: gcv = rss/m, e-bic = log(rss/m)  (Eq. (21))
    g, e = oracle.criteria(12.0, 0.0, 6, 100)
    assert g == pytest.approx(2.0) and e == pytest.approx(np.log(2.0))
    g, e = oracle.criteria(12.0, 3.0, 6, 100)  # 1 − ν/m = ½ → ×4
    assert g == pytest.approx(8.0) and e == pytest.approx(np.log(2.0) + 0.5 * (np.log(6) + np.log(100)))


def test_model_select_consistency():
    A, b = _A(4)
    x = np.zeros(40)
    x[[2, 11, 25]] = [0.5, -1.0, 0.2]
    r, nu, rss, gcv, ebic, xdb = oracle.model_select(A, b, x, 0.4)
    assert r == 3 and np.count_nonzero(xdb) <= 3 and set(np.nonzero(xdb)[0]) <= {2, 11, 25}
    assert nu == pytest.approx(oracle.dof(A, np.array([2, 11, 25]), 0.4))
    assert (gcv, ebic) == pytest.approx(oracle.criteria(rss, nu, 20, 40))
