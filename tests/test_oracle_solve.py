"""Whole-solve pins for the oracle's Algorithm 1.

References that are not the oracle: cyclic coordinate descent (textbook update,
SPEC S:541-545, licensed by P:524 "converge to the same solution"), the
Elastic Net KKT inclusion and the duality gap evaluated here in numpy, and
closed forms (orthonormal columns, single column, x = 0 above λmax, the
near-λmax single-active solution, warm start at the solution).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import synth


def cd_solve(A, b, l1, l2, tol=1e-13, max_sweeps=200000):
    """Cyclic coordinate descent on F (Eq. (1)), covariance form:
    x_j ← soft(c_j − Σ_{k≠j} G_jk x_k, λ1)/(G_jj + λ2), G = AᵀA, c = Aᵀb."""
    Acm = A.T
    G = Acm.T @ Acm
    c = Acm.T @ b
    n = G.shape[0]
    x = np.zeros(n)
    Gx = np.zeros(n)
    for _ in range(max_sweeps):
        dmax = 0.0
        for j in range(n):
            rho = c[j] - Gx[j] + G[j, j] * x[j]
            new = np.sign(rho) * max(abs(rho) - l1, 0.0) / (G[j, j] + l2)
            dj = new - x[j]
            if dj != 0.0:
                Gx += G[:, j] * dj
                x[j] = new
                dmax = max(dmax, abs(dj))
        if dmax <= tol * max(1.0, np.max(np.abs(x))):
            break
    return x


def F(A, b, x, l1, l2):
    r = A.T @ x - b
    return 0.5 * r @ r + l1 * np.abs(x).sum() + 0.5 * l2 * x @ x


def kkt_viol(A, b, x, l1, l2):
    """max_i v_i, v_i from c = Aᵀ(b − Ax) − λ2 x ∈ λ1 ∂‖x‖₁ (BASELINE north star)."""
    c = A @ (b - A.T @ x) - l2 * x
    v = np.where(x != 0, np.abs(c - l1 * np.sign(x)), np.maximum(np.abs(c) - l1, 0.0))
    return float(v.max())


def D(A, b, y, l1, l2):
    w = A @ y
    e = np.maximum(np.abs(w) - l1, 0)
    return -0.5 * y @ y - b @ y - (e @ e) / (2 * l2)


GRID = [(a, c) for a in (0.3, 0.6, 0.9) for c in (0.2, 0.5, 0.8)]


@pytest.mark.parametrize("seed", range(50))
def test_matches_coordinate_descent(seed):
    """SsNAL oracle at tol 1e-10 vs CD: ‖Δx‖∞ ≤ 1e-8‖x‖∞, same support."""
    rng = np.random.default_rng(1000 + seed)
    m = int(rng.integers(5, 21))
    n = int(rng.integers(m, 61))
    A = rng.normal(size=(n, m))
    A -= A.mean(axis=1, keepdims=True)
    A /= np.linalg.norm(A, axis=1, keepdims=True)
    xt = np.zeros(n)
    xt[rng.choice(n, 3, replace=False)] = rng.uniform(1, 2, 3) * rng.choice([-1, 1], 3)
    b = A.T @ xt + 0.1 * rng.normal(size=m)
    alpha, c = GRID[seed % len(GRID)]
    lmax = np.max(np.abs(A @ b)) / alpha
    l1, l2 = c * alpha * lmax, c * (1 - alpha) * lmax
    x, y, st, _ = oracle.solve(A, b, l1, l2, tol=1e-10)
    assert st["status"] == 0
    xc = cd_solve(A, b, l1, l2)
    scale = max(np.max(np.abs(xc)), 1e-300)
    assert np.max(np.abs(x - xc)) <= 1e-8 * scale + 1e-14
    supp_cd = np.abs(xc) > 1e-9 * scale
    supp_or = x != 0
    assert np.array_equal(supp_cd, supp_or)
    # objective agreement and certificates
    assert F(A, b, x, l1, l2) == pytest.approx(F(A, b, xc, l1, l2), rel=1e-12, abs=1e-14)
    assert st["primal_obj"] == pytest.approx(F(A, b, x, l1, l2), rel=1e-12)
    gap = F(A, b, x, l1, l2) - D(A, b, y, l1, l2)
    assert gap >= -1e-12
    # strong convexity: ‖x − x*‖ ≤ √(2 gap/λ2); gaps floored at rounding level of F
    fl = 1e-13 * max(1.0, abs(F(A, b, x, l1, l2)))
    gap_c = F(A, b, xc, l1, l2) - D(A, b, y, l1, l2)
    assert np.linalg.norm(x - xc) <= np.sqrt(2 * (max(gap, 0) + fl) / l2) + np.sqrt(2 * (max(gap_c, 0) + fl) / l2)
    assert st["dual_obj"] == pytest.approx(D(A, b, y, l1, l2), rel=1e-12, abs=1e-13)


@pytest.mark.parametrize("seed", range(5))
def test_kkt_inclusion_tight(seed):
    """At tol 1e-12 the KKT inclusion holds: max v_i ≤ 1e-9 ‖Aᵀb‖∞."""
    rng = np.random.default_rng(seed)
    m, n = 15, 50
    A = rng.normal(size=(n, m))
    b = rng.normal(size=m) * 3
    g = np.max(np.abs(A @ b))
    l1, l2 = 0.3 * g, 0.2 * g
    x, y, st, _ = oracle.solve(A, b, l1, l2, tol=1e-12)
    assert st["status"] == 0
    assert kkt_viol(A, b, x, l1, l2) <= 1e-9 * g
    assert oracle.kkt_violation(A, b, x, l1, l2) == pytest.approx(kkt_viol(A, b, x, l1, l2), abs=1e-12 * g)


@pytest.mark.parametrize("l2", [0.5, 2.0])
def test_orthonormal_closed_form(l2):
    """AᵀA = I ⇒ x* = soft(Aᵀb, λ1)/(1+λ2) (BASELINE north star)."""
    rng = np.random.default_rng(3)
    m, n = 30, 12
    Q, _ = np.linalg.qr(rng.normal(size=(m, n)))
    A = np.ascontiguousarray(Q.T)  # (n, m): columns orthonormal
    b = rng.normal(size=m) * 3
    c = A @ b
    l1 = 0.5 * np.max(np.abs(c))
    x, _, st, _ = oracle.solve(A, b, l1, l2, tol=1e-12)
    xs = np.sign(c) * np.maximum(np.abs(c) - l1, 0) / (1 + l2)
    assert np.max(np.abs(x - xs)) <= 1e-10 * np.max(np.abs(xs))


def test_single_column_closed_form():
    """n = 1: x* = soft(aᵀb, λ1)/(‖a‖² + λ2)."""
    rng = np.random.default_rng(4)
    a = rng.normal(size=(1, 9))
    b = rng.normal(size=9) * 2
    ab, aa = float(a[0] @ b), float(a[0] @ a[0])
    for l1 in (0.1 * abs(ab), 0.7 * abs(ab), 1.1 * abs(ab)):
        x, _, st, _ = oracle.solve(a, b, l1, 0.3, tol=1e-12)
        assert x[0] == pytest.approx(np.sign(ab) * max(abs(ab) - l1, 0) / (aa + 0.3), rel=1e-10, abs=1e-15)


def test_zero_above_lambda_max_one_newton_step():
    """λ1 = ‖Aᵀb‖∞ ⇒ x* = 0; under y0 = 0 exactly one Newton step."""
    cfg = synth.CONFIGS["cfg1"]
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    g = float(np.max(np.abs(oracle.aty(A, b))))
    for l1 in (g, 1.5 * g):
        x, y, st, _ = oracle.solve(A, b, l1, 0.3 * g)
        assert np.all(x == 0)
        assert st["status"] == 0 and st["newton_iters"] == 1 and st["outer_iters"] == 1
        assert st["res_kkt1"] == 0.0 and st["res_kkt3"] == 0.0
        assert np.array_equal(y, -b)


def test_near_lambda_max_single_active():
    """λ1 just below g = ‖Aᵀb‖∞: x* = e_j* soft(a_j*ᵀb, λ1)/(‖a_j*‖² + λ2) when the others stay inactive."""
    cfg = synth.CONFIGS["cfg1"]
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    c = A @ b
    j = int(np.argmax(np.abs(c)))
    g = abs(c[j])
    for eps in (1e-2, 1e-3, 1e-6):
        l1, l2 = g * (1 - eps), 0.2 * g
        xj = np.sign(c[j]) * (g - l1) / (A[j] @ A[j] + l2)
        xs = np.zeros(A.shape[0])
        xs[j] = xj
        cond = np.max(np.abs(np.delete(A @ (b - A[j] * xj), j)))
        assert cond <= l1  # closed form applies
        x, _, st, _ = oracle.solve(A, b, l1, l2, tol=1e-12)
        # error measured on the natural coefficient scale g/(‖a‖² + λ2) (tol 1e-12 run)
        assert np.max(np.abs(x - xs)) <= 1e-9 * g / (A[j] @ A[j] + l2)
        assert np.count_nonzero(x) == 1 and x[j] != 0


def test_warm_start_at_solution_zero_newton_steps():
    """x0 = x* (solved at tighter tol) ⇒ 1 outer iteration, 0 Newton steps."""
    cfg = synth.CONFIGS["cfg1"]
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    g = float(np.max(np.abs(oracle.aty(A, b))))
    l1, l2 = 0.35 * g, 0.15 * g
    xs, _, st0, _ = oracle.solve(A, b, l1, l2, tol=1e-13)
    x, _, st, _ = oracle.solve(A, b, l1, l2, tol=1e-6, x0=xs)
    assert st["outer_iters"] == 1 and st["newton_iters"] == 0 and st["aty_passes"] == 1
    assert np.max(np.abs(x - xs)) <= 1e-9 * np.max(np.abs(xs))


def test_outer_iterations_sim_like():
    """Soft pin: ≤ 6 outer iterations (allowance 8) at sim-like settings (Table 1)."""
    rng = np.random.default_rng(21)
    m, n = 100, 10_000
    A = rng.normal(size=(n, m))
    xt = np.zeros(n)
    sup = rng.choice(n, 20, replace=False)
    xt[sup] = 5.0
    s = A.T @ xt
    b = s + rng.normal(size=m) * np.sqrt(s.var() / 5)
    for alpha in (0.6, 0.9):
        lmax = np.max(np.abs(A @ b)) / alpha
        x, _, st, _ = oracle.solve(A, b, 0.5 * alpha * lmax, 0.5 * (1 - alpha) * lmax)
        assert st["status"] == 0
        assert st["outer_iters"] <= 8
        # σ schedule: σ0 × 5^(outer−1)
        assert st["sigma_final"] == pytest.approx(5e-3 * 5.0 ** (st["outer_iters"] - 1))


def test_thread_count_invariance():
    """Results are bit-identical for 1 and 8 OpenMP threads (fixed summation order)."""
    code = (
        "import numpy as np, oracle, synth;"
        "c=synth.scaled(synth.CONFIGS['cfg2'], n=3000);A=synth.design(c);b,_=synth.response(c);"
        "g=float(np.max(np.abs(oracle.aty(A,b))));x,y,st,_=oracle.solve(A,b,0.3*g,0.1*g);"
        "import sys;sys.stdout.write(x.tobytes().hex()[:4000]+str(st['newton_iters']))"
    )
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for th in ("1", "8"):
        env = dict(os.environ, OMP_NUM_THREADS=th, PYTHONPATH=root)
        outs.append(subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                                   check=True).stdout)
    assert outs[0] == outs[1]
