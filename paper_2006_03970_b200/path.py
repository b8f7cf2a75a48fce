"""λ path with warm starts, a max-active cap and model selection (Section 3.3).

Orchestration only: every solve and every criterion (ν, OLS de-biasing, rss, GCV, e-BIC) is
computed by the C-ABI (ssnal_en_solve / ssnal_en_model_select); this module loops over the grid
and picks the minimiser of each criterion.
"""
from __future__ import annotations

import math

import numpy as np


def lambda_grid(n_points: int = 100, c_max: float = 1.0, c_min: float = 0.1) -> np.ndarray:
    """Log-spaced c values from c_max down to c_min (Table D.4 protocol: 100 points, 1 → 0.1)."""
    return np.logspace(math.log10(c_max), math.log10(c_min), n_points)


def solve_path(P, alpha: float, cs, sigma0: float = 5e-3, tol: float = 1e-6, max_active: int | None = None,
               select: bool = True, debias: bool = False, carry_sigma: bool = True, carry_dual: bool = True):
    """Solve along c ∈ cs with λ1 = c α λmax, λ2 = c (1 − α) λmax, λmax = ‖Aᵀb‖∞/α,
    warm-starting each point at the previous solution and — reading R38 — at the
    previous point's final σ (carry_sigma; False restarts every point at σ0) and — reading R39 — at its
    final dual iterate (carry_dual: option warm_dual for every point after the first, so the warm start
    costs no Aᵀ pass; the handle keeps y and w between the calls).  The path stops once a
    solution has at least `max_active` nonzeros.  Returns (points, best) where best maps
    'gcv' / 'ebic' to the index of the minimising point (None without selection)."""
    lmax = P.lambda_max_l1 / alpha
    points = []
    x = None
    sig = sigma0
    for i, c in enumerate(cs):
        l1, l2 = c * alpha * lmax, c * (1 - alpha) * lmax
        P.set_option("warm_dual", 1 if (carry_dual and i > 0) else 0)
        x, st = P.solve(l1, l2, sig, tol, x0=x)
        if carry_sigma:
            sig = st["sigma_final"]
        crit, xdb = P.model_select(l2, debias) if select else (None, None)
        points.append({"c": float(c), "lambda1": l1, "lambda2": l2, "x": x, "stats": st, "criteria": crit,
                       "x_debiased": xdb})
        if max_active is not None and st["active"] >= max_active:
            break
    P.set_option("warm_dual", 0)
    best = {}
    if select:
        for key in ("gcv", "ebic"):
            vals = [p["criteria"][key] for p in points]
            finite = [i for i, v in enumerate(vals) if v == v]
            best[key] = min(finite, key=lambda i: vals[i]) if finite else None
    return points, best


def cv_path(make_problem, m: int, alpha: float, cs, lambda_max_l1: float, k: int = 5, sigma0: float = 5e-3,
            tol: float = 1e-6, carry_dual: bool = True):
    """k-fold cross-validation along the path (Section 3.3; reading R35).

    make_problem(rows) must return a Problem over the given rows of (A, b) (e.g. a handle created
    from a row subset in device memory).  Folds are interleaved (row r in fold r mod k); the grid
    uses the full-data λmax = lambda_max_l1/α for every fold.  Each fold solves the
    warm-started path on its training rows (σ carried along the path, reading R38); the held-out error ‖b_test − A_test x‖² is computed by
    the test handle (ssnal_en_residual).  Returns (cv, best) with cv[i] = Σ_folds err / m."""
    lmax = lambda_max_l1 / alpha
    cv = np.zeros(len(cs))
    for f in range(k):
        test = np.arange(f, m, k)
        train = np.setdiff1d(np.arange(m), test)
        Ptr, Pte = make_problem(train), make_problem(test)
        try:
            x = None
            sig = sigma0
            for i, c in enumerate(cs):
                l1, l2 = c * alpha * lmax, c * (1 - alpha) * lmax
                Ptr.set_option("warm_dual", 1 if (carry_dual and i > 0) else 0)  # reading R39
                x, st = Ptr.solve(l1, l2, sig, tol, x0=x)
                sig = st["sigma_final"]  # reading R38
                cv[i] += Pte.residual(x)
        finally:
            Ptr.close()
            Pte.close()
    cv /= m
    return cv, int(np.argmin(cv))
