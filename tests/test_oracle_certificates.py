"""Pins of the oracle's certificates and of its fused K1-equivalent (test infrastructure only).

* orc_primal_obj, orc_kkt_violation, orc_dual_obj: hand-evaluated values on a 2 x 3 integer problem
  (tests/golden/certificate_examples.txt, every line derived there), including a point with a zero
  duality gap (x* = (0, 0, ½) with y* = Ax* − b: strong duality, P:113-125 and (D) P:209), and the
  orthonormal-design closed form x* = soft(Aᵀb, λ1)/(1 + λ2) (BASELINE north star) where the KKT
  violation vanishes and the gap closes; the whole solve reproduces the hand-derived minimiser.
* orc_aty_fused (the reference of the K1/K1g parity tests) against the separately pinned pieces:
  orc_aty (w), orc_active_set (J, Eq. (17)), orc_prox (P_J, Eq. (6)), orc_grad_psi (g, Eq. (15)),
  and a numpy evaluation of the four partial sums from their definitions, incl. exact ties
  |t_i| = σλ1 (strict '>' of P:354, R11) and both signs of t.
"""
import os

import numpy as np
import pytest

import oracle
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "certificate_examples.txt")
A23 = np.array([[1.0, 0.0], [0.0, 1.0], [2.0, -1.0]])  # (n, m): rows are the columns a1, a2, a3
B23 = np.array([3.0, 1.0])
L1, L2 = 2.0, 1.0


def _rows():
    out = []
    for line in open(GOLDEN):
        if line.startswith("#") or not line.strip():
            continue
        f = line.split()
        out.append((f[0], [float(v) for v in f[1:4] if v != "-"], float(f[4]), " ".join(f[5:])))
    return out


@pytest.mark.parametrize("row", _rows(), ids=lambda r: f"{r[0]}{r[1]}")
def test_certificate_golden(row):
    kind, v, expected, why = row
    if kind == "primal":
        got = oracle.primal_obj(A23, B23, np.array(v), L1, L2)
    elif kind == "kkt":
        got = oracle.kkt_violation(A23, B23, np.array(v), L1, L2)
    else:
        y = np.array(v)
        got = oracle.dual_obj(B23, y, oracle.aty(A23, y), L1, L2)
    assert got == expected, (row, got)  # integer data: exact in fp64


def test_solve_reaches_hand_derived_minimiser():
    """x* = (0, 0, ½) (derived in the golden file: single-column closed form on a3, the other two
    columns inside the λ1 box) — the iteration must land on it, with a vanishing gap."""
    x, y, st, _ = oracle.solve(A23, B23, L1, L2, tol=1e-12)
    np.testing.assert_allclose(x, [0.0, 0.0, 0.5], atol=1e-12)
    np.testing.assert_allclose(y, [-2.0, -1.5], atol=1e-11)
    assert st["gap"] == pytest.approx(0.0, abs=1e-11) and st["primal_obj"] == pytest.approx(4.25, rel=1e-13)


def test_orthonormal_closed_form_certificates():
    """Orthonormal columns (AᵀA = I): x* = soft(Aᵀb, λ1)/(1 + λ2) (BASELINE north star).  There the KKT
    violation is at roundoff level, D(Ax* − b) = F(x*), and any perturbation raises both."""
    rng = np.random.default_rng(11)
    m, n = 40, 12
    Q, _ = np.linalg.qr(rng.standard_normal((m, n)))
    A = np.ascontiguousarray(Q.T)
    b = rng.standard_normal(m) * 3
    c = Q.T @ b
    l1, l2 = 0.5 * np.max(np.abs(c)), 0.7
    xs = np.sign(c) * np.maximum(np.abs(c) - l1, 0) / (1 + l2)
    assert 0 < np.count_nonzero(xs) < n
    assert oracle.kkt_violation(A, b, xs, l1, l2) <= 1e-13 * np.max(np.abs(c))
    F = oracle.primal_obj(A, b, xs, l1, l2)
    y = Q @ xs - b
    D = oracle.dual_obj(b, y, oracle.aty(A, y), l1, l2)
    assert abs(F - D) <= 1e-13 * abs(F)
    xp = xs.copy()
    xp[np.argmax(np.abs(xs))] *= 1.01
    assert oracle.kkt_violation(A, b, xp, l1, l2) > 1e-4
    assert oracle.primal_obj(A, b, xp, l1, l2) > F


@pytest.mark.parametrize("sigma", [1.0, 0.37])
def test_aty_fused_matches_pinned_pieces(sigma):
    cfg = synth.scaled(synth.CONFIGS["cfg3"], n=3000, m=37)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    y = synth.normals(21, 1, cfg.m)
    x = np.zeros(cfg.n)
    x[::7] = synth.normals(21, 2, len(x[::7]))
    w_ref = oracle.aty(A, y)
    t = x - sigma * w_ref
    l2 = 0.3
    l1 = float(np.quantile(np.abs(t), 0.9)) / sigma
    if sigma == 1.0:  # exact ties |t_i| = σλ1 (σ = 1 so σλ1 == λ1 bitwise): inactive, P = 0
        l1 = float(np.sort(np.abs(t))[int(0.9 * cfg.n)])
        tie = np.abs(t) == sigma * l1
        assert tie.sum() >= 1
    w, J, PJ, part, g = oracle.aty_fused(A, b, y, x, sigma, l1, l2)
    assert np.array_equal(w, w_ref)
    assert np.array_equal(J, oracle.active_set(t, sigma, l1))
    assert np.array_equal(PJ, oracle.prox(t[J], sigma, l1, l2))
    assert np.any(t[J] > 0) and np.any(t[J] < 0)
    # the four partial sums from their definitions, evaluated independently in numpy
    thr = sigma * l1
    P = np.where(np.abs(t) > thr, np.sign(t) * (np.abs(t) - thr) / (1 + sigma * l2), 0.0)
    z = (x - P) / sigma - w_ref
    ref = [P @ P, (x - P) @ (x - P), z @ z, np.sum(np.maximum(np.abs(w_ref) - l1, 0.0) ** 2)]
    np.testing.assert_allclose(part, ref, rtol=1e-12)
    # p*(Aᵀy) of Prop. 1 is partial[3]/(2λ2)
    assert part[3] / (2 * l2) == pytest.approx(oracle.pstar(w_ref, l1, l2), rel=1e-12)
    # g = y + b − A_J P_J equals the pinned ∇ψ (Eq. (15)) bitwise (same order) and numpy to 1e-12
    assert np.array_equal(g, oracle.grad_psi(A, b, x, y, sigma, l1, l2))
    np.testing.assert_allclose(g, y + b - A[J].T @ PJ, rtol=0, atol=1e-12 * (1 + np.abs(g).max()))


def test_aty_fused_empty_and_full_active_sets():
    cfg = synth.scaled(synth.CONFIGS["cfg1"], n=200)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    y = synth.normals(22, 1, cfg.m)
    x = np.zeros(cfg.n)
    _, J, PJ, part, g = oracle.aty_fused(A, b, y, x, 1.0, 1e30, 0.5)  # nothing active: g = y + b
    assert len(J) == 0 and part[0] == 0.0 and np.array_equal(g, y + b)
    _, J, PJ, part, g = oracle.aty_fused(A, b, y, x, 1.0, 0.0, 0.5)  # λ1 = 0: all t_i ≠ 0 active
    w = oracle.aty(A, y)
    assert np.array_equal(J, np.nonzero(w != 0)[0])
    np.testing.assert_allclose(PJ, -w[J] / 1.5, rtol=1e-15)
