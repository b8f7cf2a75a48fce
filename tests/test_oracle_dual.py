"""Pins for the oracle's Section 3 pieces: h*, ψ (Prop. 2), ∇ψ (Eq. (15)), z̄, the
multiplier update and the active set / Newton system (Eq. (16)-(19)).

Independent references used here: the augmented Lagrangian Eq. (7) evaluated
term by term, its minimisation over z done numerically, central
finite differences, and dense numpy linear algebra on V = I + σ A Q Aᵀ with Q
built from its definition Eq. (17).
"""
import numpy as np
import pytest
from scipy.optimize import minimize

import oracle


def _inst(seed, m=7, n=19, scale_x=1.0):
    rng = np.random.default_rng(seed)
    A = rng.normal(size=(n, m))  # (n, m) = column-major m x n
    b = rng.normal(size=m) * 2
    x = rng.normal(size=n) * scale_x * (rng.random(n) < 0.4)
    y = rng.normal(size=m)
    sigma, l1, l2 = rng.uniform(0.2, 2), rng.uniform(0.3, 2), rng.uniform(0.1, 2)
    return A, b, x, y, sigma, l1, l2


def _pstar_np(z, l1, l2):  # Prop. 1, used only inside the L_sigma reference below
    e = np.maximum(np.abs(z) - l1, 0.0)
    return float(np.sum(e * e) / (2 * l2))


def _L_sigma(A, b, x, y, z, sigma, l1, l2):
    """Eq. (7): h*(y) + p*(z) − xᵀ(Aᵀy + z) + σ/2 ‖Aᵀy + z‖²."""
    r = A @ y + z  # (n,m)@(m,) = Aᵀy in column-major terms
    return 0.5 * y @ y + b @ y + _pstar_np(z, l1, l2) - x @ r + 0.5 * sigma * r @ r


def test_hstar_examples():
    assert oracle.hstar(np.zeros(3), np.array([1.0, 2, 3])) == 0.0
    assert oracle.hstar(np.array([1.0, 1.0]), np.array([2.0, -1.0])) == 2.0
    b = np.array([1.5, -2.0, 0.25])
    assert oracle.hstar(-b, b) == pytest.approx(-0.5 * b @ b)


@pytest.mark.parametrize("seed", range(8))
def test_psi_equals_L_sigma_at_zbar(seed):
    """Prop. 2: ψ(y) = L_σ(y, z̄; x) with z̄ = argmin_z L_σ(y, z; x)."""
    A, b, x, y, sigma, l1, l2 = _inst(seed)
    zb = oracle.zbar(A, x, y, sigma, l1, l2)
    psi = oracle.psi(A, b, x, y, sigma, l1, l2)
    ref = _L_sigma(A, b, x, y, zb, sigma, l1, l2)
    assert psi == pytest.approx(ref, rel=1e-13, abs=1e-13)
    # z̄ is the minimiser of L_σ(y, ·; x): numerical minimisation cannot do better
    f = lambda z: _L_sigma(A, b, x, y, z, sigma, l1, l2)
    res = minimize(f, np.zeros_like(zb), method="BFGS", options={"gtol": 1e-10})
    assert f(zb) <= res.fun + 1e-9
    assert np.max(np.abs(res.x - zb)) < 1e-4


def test_psi_zero_state():
    """x = 0, y = 0 → ψ = 0; ∇ψ = b."""
    A, b, x, y, sigma, l1, l2 = _inst(3)
    assert oracle.psi(A, b, np.zeros_like(x), np.zeros_like(y), sigma, l1, l2) == 0.0
    g = oracle.grad_psi(A, b, np.zeros_like(x), np.zeros_like(y), sigma, l1, l2)
    assert np.array_equal(g, b)


@pytest.mark.parametrize("seed", range(6))
def test_grad_psi_finite_differences(seed):
    """Eq. (15) with ∇h* = y + b (R1) vs central differences of ψ."""
    A, b, x, y, sigma, l1, l2 = _inst(seed, m=6, n=25)
    g = oracle.grad_psi(A, b, x, y, sigma, l1, l2)
    h = 1e-6
    fd = np.empty_like(g)
    for k in range(len(y)):
        e = np.zeros_like(y)
        e[k] = h
        fd[k] = (oracle.psi(A, b, x, y + e, sigma, l1, l2) - oracle.psi(A, b, x, y - e, sigma, l1, l2)) / (2 * h)
    assert np.max(np.abs(fd - g)) <= 1e-6 * max(1.0, np.max(np.abs(g)))
    # the y − b variant printed at P:226 must NOT match (reading R1)
    assert np.max(np.abs(fd - (g - 2 * b))) > 1e-3


def test_grad_inside_box():
    """If x − σAᵀy lies inside the σλ1 box, ∇ψ(y) = y + b."""
    A, b, x, y, sigma, l1, l2 = _inst(4)
    x = np.zeros_like(x)
    y = y * 1e-6
    l1 = 1e3
    assert np.allclose(oracle.grad_psi(A, b, x, y, sigma, l1, l2), y + b, rtol=0, atol=1e-15)


def test_psi_convex():
    """ψ is convex along random segments."""
    A, b, x, y, sigma, l1, l2 = _inst(5, m=5, n=30, scale_x=3)
    rng = np.random.default_rng(1)
    for _ in range(50):
        y1, y2 = rng.normal(size=5) * 3, rng.normal(size=5) * 3
        t = rng.random()
        lhs = oracle.psi(A, b, x, t * y1 + (1 - t) * y2, sigma, l1, l2)
        rhs = t * oracle.psi(A, b, x, y1, sigma, l1, l2) + (1 - t) * oracle.psi(A, b, x, y2, sigma, l1, l2)
        assert lhs <= rhs + 1e-10


def test_zbar_scalar_and_moreau():
    """z update scalar example and the Moreau form z̄ = (t − prox(t))/σ."""
    A = np.array([[1.0]])
    z = oracle.zbar(A, np.array([3.0]), np.array([0.0]), 1.0, 1.0, 1.0)
    assert z[0] == 2.0
    A, b, x, y, sigma, l1, l2 = _inst(6)
    t = x - sigma * (A @ y)
    zb = oracle.zbar(A, x, y, sigma, l1, l2)
    assert np.allclose(zb, (t - oracle.prox(t, sigma, l1, l2)) / sigma, rtol=1e-12, atol=1e-12)


def test_multiplier_update_equals_prox():
    """x − σ(Aᵀy + z̄) = prox_{σp}(x − σAᵀy) (Eq. (10) with Prop. 2(2); used as x ← P)."""
    for seed in range(5):
        A, b, x, y, sigma, l1, l2 = _inst(seed)
        w = A @ y
        zb = oracle.zbar(A, x, y, sigma, l1, l2)
        xnew = x - sigma * (w + zb)
        P = oracle.prox(x - sigma * w, sigma, l1, l2)
        assert np.allclose(xnew, P, rtol=1e-12, atol=1e-12)
    # S:164 hand value: σ=2, x=1, Aᵀy+z = 0.25 → 0.5
    assert 1.0 - 2.0 * 0.25 == 0.5


def test_dual_objective_is_lower_bound():
    """Weak duality: F(x) ≥ D(y) = −h*(y) − p*(Aᵀy) for arbitrary x, y (reading R2)."""
    rng = np.random.default_rng(12)
    A, b, _, _, _, l1, l2 = _inst(12, m=8, n=30)
    for _ in range(100):
        x = rng.normal(size=30) * (rng.random(30) < 0.3)
        y = rng.normal(size=8) * 2
        F = oracle.primal_obj(A, b, x, l1, l2)
        D = oracle.dual_obj(b, y, A @ y, l1, l2)
        assert F >= D - 1e-12


# ---------------- active set and Newton system -------------------------------


def test_active_set_example():
    """σ = λ1 = 1, t = (3, 0.5, −2) → J = {1, 3} (1-based), r = 2 (Eq. (17))."""
    J = oracle.active_set(np.array([3.0, 0.5, -2.0]), 1.0, 1.0)
    assert list(J) == [0, 2]
    assert len(oracle.active_set(np.array([0.2, -0.3]), 1.0, 1.0)) == 0
    assert list(oracle.active_set(np.array([1.0, -1.0, 1.0000001]), 1.0, 1.0)) == [2]  # ties inactive (R11)


def _dense_newton(A, x, y, sigma, l1, l2, b):
    """V = I_m + σ A Q Aᵀ with Q diagonal from Eq. (17); d = −V⁻¹∇ψ via LU."""
    Acm = A.T  # m x n
    t = x - sigma * (A @ y)
    q = np.where(np.abs(t) > sigma * l1, 1.0 / (1.0 + sigma * l2), 0.0)
    V = np.eye(Acm.shape[0]) + sigma * (Acm * q) @ Acm.T
    g = oracle.grad_psi(A, b, x, y, sigma, l1, l2)
    return np.linalg.solve(V, -g), g, np.nonzero(np.abs(t) > sigma * l1)[0]


@pytest.mark.parametrize("case", ["smw", "mxm", "empty"])
def test_newton_direction_vs_dense(case):
    """Eq. (18) (r ≥ m) and SMW Eq. (19) (r < m) agree with a dense solve of V d = −∇ψ to 1e-10."""
    rng = np.random.default_rng({"smw": 1, "mxm": 2, "empty": 3}[case])
    m, n = 12, 40
    A = rng.normal(size=(n, m))
    b = rng.normal(size=m)
    x = rng.normal(size=n) * (rng.random(n) < 0.5)
    y = rng.normal(size=m)
    sigma, l2 = 0.7, 0.4
    w = A @ y
    mag = np.sort(np.abs(x - sigma * w))[::-1]
    r_target = {"smw": 5, "mxm": 25, "empty": 0}[case]
    # choose λ1 so that exactly r_target entries are active
    thr = (mag[r_target - 1] + mag[r_target]) / 2 if r_target > 0 else mag[0] * 1.01
    l1 = thr / sigma
    d_ref, g, J = _dense_newton(A, x, y, sigma, l1, l2, b)
    assert len(J) == r_target
    kappa = sigma / (1 + sigma * l2)
    d, br = oracle.newton_direction(A, J, g, kappa)
    assert br == {"smw": 1, "mxm": 2, "empty": 0}[case]
    assert np.max(np.abs(d - d_ref)) <= 1e-10 * max(1.0, np.max(np.abs(d_ref)))
    if np.any(g):
        assert g @ d < 0  # descent


def test_sigma_AQAt_equals_kappa_AJAJt():
    """σ A Q Aᵀ = κ A_J A_Jᵀ."""
    rng = np.random.default_rng(4)
    m, n = 6, 20
    A = rng.normal(size=(n, m))
    t = rng.normal(size=n) * 2
    sigma, l1, l2 = 0.9, 0.8, 0.3
    q = np.where(np.abs(t) > sigma * l1, 1 / (1 + sigma * l2), 0.0)
    J = oracle.active_set(t, sigma, l1)
    kappa = sigma / (1 + sigma * l2)
    lhs = sigma * (A.T * q) @ A
    rhs = kappa * A[J].T @ A[J]
    assert np.allclose(lhs, rhs, rtol=1e-14, atol=1e-14)
    assert 1.0 / (1.0 + 1.0 * 1.0) == 0.5  # σ=1, λ2=1 → κ = 1/2


def test_chol_vs_numpy():
    rng = np.random.default_rng(0)
    for N in (1, 2, 7, 33):
        B = rng.normal(size=(N, N))
        M = B @ B.T + N * np.eye(N)
        L = oracle.chol(M)
        assert np.allclose(L, np.linalg.cholesky(M), rtol=1e-12, atol=1e-12)
    with pytest.raises(FloatingPointError):
        oracle.chol(np.array([[1.0, 2.0], [2.0, 1.0]]))
