"""Pins for the oracle's conjugate-gradient Newton direction (Algorithm 1 step (1), P:273;
P:379; reading R32: textbook CG from d0 = 0, stop at ‖Vd + g‖ ≤ tol‖g‖).

What fixes CG independently of its own code:
  * V = I + κA_JA_Jᵀ with k distinct eigenvalues → exact termination in ≤ k iterations (Krylov
    dimension), at the closed forms of Sherman–Morrison (r = 1) and of orthonormal columns;
  * a dense solve of the same V (np.linalg.solve) within the requested tolerance;
  * every CG iterate from d0 = 0 is a descent direction (gᵀd < 0);
  * the CG strategy inside the whole solve reaches the same minimiser as the exact branches.
"""
import numpy as np
import pytest

import oracle
import synth


def V_of(A, J, kappa):
    AJ = A[J].T  # m × r (A is (n, m): row i is column a_i)
    return np.eye(A.shape[1]) + kappa * AJ @ AJ.T


@pytest.mark.parametrize("m,n,step,kappa,seed", [(30, 200, 3, 0.7, 0), (12, 40, 1, 5.0, 1), (50, 60, 7, 1e-3, 2)])
def test_cg_matches_dense_solve(m, n, step, kappa, seed):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((n, m))
    J = np.arange(0, n, step)
    g = rng.standard_normal(m)
    d, it = oracle.cg_direction(A, J, g, kappa, tol=1e-13)
    ref = np.linalg.solve(V_of(A, J, kappa), -g)
    assert np.linalg.norm(d - ref) <= 1e-11 * np.linalg.norm(ref)
    assert it <= 4 * m  # finite termination up to rounding


def test_rank_one_terminates_in_two_iterations_sherman_morrison():
    """r = 1: V = I + κaaᵀ has two distinct eigenvalues → 2 CG iterations; d by Sherman–Morrison."""
    rng = np.random.default_rng(3)
    m = 40
    A = rng.standard_normal((5, m))
    J = np.array([2])
    g = rng.standard_normal(m)
    kappa = 0.37
    d, it = oracle.cg_direction(A, J, g, kappa, tol=1e-14)
    a = A[2]
    closed = -g + kappa * a * (a @ g) / (1.0 + kappa * (a @ a))
    assert it <= 2
    assert np.allclose(d, closed, rtol=1e-12, atol=1e-14)


def test_orthonormal_columns_two_eigenvalues():
    """A_J with orthonormal columns: V has eigenvalues {1, 1+κ} → ≤ 2 iterations,
    d = −g + κ/(1+κ) A_J A_Jᵀ g."""
    rng = np.random.default_rng(4)
    m, r = 25, 6
    Q, _ = np.linalg.qr(rng.standard_normal((m, r)))
    A = np.vstack([rng.standard_normal((3, m)), Q.T])  # columns 3..8 are orthonormal
    J = np.arange(3, 3 + r)
    g = rng.standard_normal(m)
    kappa = 2.5
    d, it = oracle.cg_direction(A, J, g, kappa, tol=1e-14)
    closed = -g + kappa / (1.0 + kappa) * Q @ (Q.T @ g)
    assert it <= 2
    assert np.allclose(d, closed, rtol=1e-12, atol=1e-14)


def test_empty_set_and_identity():
    rng = np.random.default_rng(5)
    A = rng.standard_normal((10, 8))
    g = rng.standard_normal(8)
    d, it = oracle.cg_direction(A, np.zeros(0, dtype=np.int64), g, 0.9, tol=1e-14)
    assert it == 1 and np.allclose(d, -g, rtol=0, atol=1e-15)


@pytest.mark.parametrize("maxit", [1, 2, 3, 5])
def test_every_iterate_is_descent(maxit):
    rng = np.random.default_rng(6)
    m = 20
    A = rng.standard_normal((60, m))
    J = np.arange(0, 60, 2)
    g = rng.standard_normal(m)
    d, it = oracle.cg_direction(A, J, g, 3.0, tol=1e-30, maxit=maxit)
    assert it == maxit
    assert g @ d < 0
    # the residual decreases in the V⁻¹ norm: the error energy is below that of d = 0
    V = V_of(A, J, 3.0)
    e = d - np.linalg.solve(V, -g)
    e0 = np.linalg.solve(V, -g)
    assert e @ V @ e < e0 @ V @ e0


def test_cg_equals_exact_branch_to_tolerance():
    """The exact branches (Eq. (18)/(19)) and CG agree to the CG tolerance."""
    rng = np.random.default_rng(7)
    m = 30
    A = rng.standard_normal((400, m))
    for J in (np.arange(0, 400, 40), np.arange(0, 400, 2)):  # r < m (SMW) and r ≥ m (m × m)
        g = rng.standard_normal(m)
        d_exact, br = oracle.newton_direction(A, J, g, 0.8)
        d_cg, _ = oracle.cg_direction(A, J, g, 0.8, tol=1e-13)
        assert br in (1, 2)
        assert np.linalg.norm(d_cg - d_exact) <= 1e-10 * np.linalg.norm(d_exact)


def test_solve_with_cg_strategy_reaches_the_same_minimiser():
    """Algorithm 1 with every Newton system solved by CG (cg_ratio small) reaches the exact
    branches' minimiser (strong convexity: unique x*), with the same outer iterations."""
    cfg = synth.CONFIGS["cfg1"]
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    lm = float(np.max(np.abs(oracle.aty(A, b)))) / cfg.alpha
    l1, l2 = 0.3 * cfg.alpha * lm, 0.3 * (1 - cfg.alpha) * lm
    x0, _, s0, _ = oracle.solve(A, b, l1, l2)
    x1, _, s1, _ = oracle.solve(A, b, l1, l2, cg_ratio=1e-9)
    assert s0["status"] == 0 and s1["status"] == 0
    assert s1["branch_steps"][3] > 0 and s1["branch_steps"][1] == s1["branch_steps"][2] == 0
    assert s1["cg_iters"] >= s1["branch_steps"][3]
    F0 = oracle.primal_obj(A, b, x0, l1, l2)
    F1 = oracle.primal_obj(A, b, x1, l1, l2)
    assert abs(F1 - F0) <= 1e-10 * abs(F0)
    assert np.max(np.abs(x1 - x0)) <= 1e-6 * np.max(np.abs(x0))
    assert s1["outer_iters"] == s0["outer_iters"]
    # the paper's rule alone (min(m, r) > 10⁴) never selects CG at m = 50
    _, _, s2, _ = oracle.solve(A, b, l1, l2, cg_threshold=1e4)
    assert s2["branch_steps"][3] == 0
