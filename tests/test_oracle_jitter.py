"""Pins for the oracle's factor retry ("factorization failure (numerically non-SPD) → ...
caller retries with jitter 1e−10·I"; SURVEY §8(b) SSNAL_ENUMERIC; reading R36: the retry scales
the diagonal of the factored matrix by (1 + jitter)).

V = I + κA_JA_Jᵀ ⪰ I is SPD in exact arithmetic, so a pivot failure needs roundoff of the order
of the smallest pivot: duplicated columns make A_JA_Jᵀ (m × m branch) and A_JᵀA_J (SMW branch)
rank one, and κ = 1e20-1e25 puts the cancellation error (ε κ‖a‖²) far above the pivots that
remain.  The jittered factor must then succeed and the direction must solve the jittered system,
checked against numpy's LAPACK solve of that system written out independently here."""
import numpy as np
import pytest

import oracle


def dup_case(m=6, r=12, seed=1):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal(m)
    A = np.ascontiguousarray(np.tile(a, (r, 1)))  # (n, m): every column equal to a
    g = rng.standard_normal(m)
    return A, g


@pytest.mark.parametrize("kappa", [1e20, 1e25])
def test_mm_branch_fails_then_solves_jittered_system(kappa):
    A, g = dup_case()
    m, r = A.shape[1], A.shape[0]
    J = np.arange(r)
    with pytest.raises(FloatingPointError):
        oracle.newton_direction(A, J, g, kappa)
    d, br = oracle.newton_direction(A, J, g, kappa, jitter=1e-10)
    assert br == 2
    M = np.eye(m) + kappa * A.T @ A  # A.T is m × r = A_J
    M[np.diag_indices(m)] *= 1.0 + 1e-10
    # backward-stable solve: small residual relative to ‖M‖‖d‖
    assert np.linalg.norm(M @ d + g) <= 1e-12 * np.linalg.norm(M, 2) * np.linalg.norm(d)
    d_np = np.linalg.solve(M, -g)
    assert np.linalg.norm(d - d_np) <= 1e-4 * np.linalg.norm(d_np)
    assert g @ d < 0  # still a descent direction


@pytest.mark.parametrize("kappa", [1e20, 1e25])
def test_smw_branch_fails_then_solves_jittered_system(kappa):
    A, g = dup_case(m=8, r=3, seed=2)
    J = np.arange(3)
    with pytest.raises(FloatingPointError):
        oracle.newton_direction(A, J, g, kappa)
    d, br = oracle.newton_direction(A, J, g, kappa, jitter=1e-10)
    assert br == 1
    AJ = A.T  # m × r
    Gj = np.eye(3) / kappa + AJ.T @ AJ
    Gj[np.diag_indices(3)] *= 1.0 + 1e-10
    d_np = -g + AJ @ np.linalg.solve(Gj, AJ.T @ g)
    assert np.linalg.norm(d - d_np) <= 1e-4 * np.linalg.norm(g)
    assert g @ d < 0


def test_zero_jitter_is_the_plain_direction():
    """jitter = 0 leaves Eq. (18)/(19) unchanged (bitwise: the same arithmetic)."""
    rng = np.random.default_rng(3)
    A = rng.standard_normal((30, 10))
    g = rng.standard_normal(10)
    for J in (np.arange(4), np.arange(25)):
        d0, b0 = oracle.newton_direction(A, J, g, 0.7)
        d1, b1 = oracle.newton_direction(A, J, g, 0.7, jitter=0.0)
        assert b0 == b1 and np.array_equal(d0, d1)
        # and a small jitter on a well-conditioned system moves d by O(jitter)
        d2, _ = oracle.newton_direction(A, J, g, 0.7, jitter=1e-10)
        assert 0 < np.max(np.abs(d2 - d0)) <= 1e-8 * np.max(np.abs(d0))
