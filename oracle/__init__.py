"""CPU oracle for SsNAL-EN — TEST INFRASTRUCTURE ONLY.

Thin ctypes wrapper around libssnal_oracle.so (oracle/ssnal_oracle.c), the
plain fp64 C implementation of the paper's method.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this module; the product package never does.  Shares no code with the
CUDA path.

Arrays: A is a C-contiguous float64 array of shape (n, m) (= column-major m x n,
column i is A[i]).  Parity status of every function is listed in DESIGN.md
("Oracle pins"); none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(_HERE, "libssnal_oracle.so")
_lib = None

_d = ctypes.c_double
_i64 = ctypes.c_int64
_dp = ctypes.POINTER(ctypes.c_double)
_lp = ctypes.POINTER(ctypes.c_int64)


class Opts(ctypes.Structure):
    _fields_ = [("sigma_factor", _d), ("sigma_max", _d), ("mu", _d), ("beta", _d), ("max_outer", ctypes.c_int32),
                ("max_inner", ctypes.c_int32), ("max_bt", ctypes.c_int32), ("init_mode", ctypes.c_int32),
                ("cg_ratio", _d), ("cg_threshold", _d), ("cg_tol", _d), ("cg_maxit", ctypes.c_int32),
                ("inner_tol_mode", ctypes.c_int32), ("jitter", _d)]


class Stats(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("outer_iters", ctypes.c_int32), ("newton_iters", ctypes.c_int32),
                ("backtracks", ctypes.c_int32), ("aty_passes", ctypes.c_int32),
                ("branch_steps", ctypes.c_int32 * 4), ("line_search_stalled", ctypes.c_int32),
                ("cg_iters", ctypes.c_int32), ("jitter_retries", ctypes.c_int32), ("active", ctypes.c_int64), ("res_kkt1", _d), ("res_kkt3", _d), ("primal_obj", _d),
                ("dual_obj", _d), ("gap", _d), ("sigma_final", _d)]


class Trace(ctypes.Structure):
    _fields_ = [("outer", ctypes.c_int32), ("branch", ctypes.c_int32), ("r", ctypes.c_int64), ("s", _d),
                ("psi", _d), ("res1", _d), ("gd", _d), ("jsum", ctypes.c_int64)]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise RuntimeError(f"{LIB} missing: run tools/build.py")
        L = ctypes.CDLL(LIB)
        sig = {
            "orc_penalty": (_d, [_dp, _i64, _d, _d]),
            "orc_pstar": (_d, [_dp, _i64, _d, _d]),
            "orc_prox": (_d, [_d, _d, _d, _d]),
            "orc_prox_conj": (_d, [_d, _d, _d, _d]),
            "orc_hstar": (_d, [_dp, _dp, _i64]),
            "orc_aty": (None, [_dp, _i64, _i64, _dp, _dp]),
            "orc_ax": (None, [_dp, _i64, _i64, _dp, _dp]),
            "orc_psi": (_d, [_dp, _dp, _i64, _i64, _dp, _dp, _d, _d, _d]),
            "orc_grad_psi": (None, [_dp, _dp, _i64, _i64, _dp, _dp, _d, _d, _d, _dp]),
            "orc_zbar": (None, [_dp, _i64, _i64, _dp, _dp, _d, _d, _d, _dp]),
            "orc_active_set": (_i64, [_dp, _i64, _d, _d, _lp]),
            "orc_chol": (ctypes.c_int, [_dp, _i64]),
            "orc_chol_solve": (None, [_dp, _i64, _dp]),
            "orc_newton_direction": (ctypes.c_int, [_dp, _i64, _lp, _i64, _dp, _d, _d, _dp]),
            "orc_cg_direction": (ctypes.c_int, [_dp, _i64, _lp, _i64, _dp, _d, _d, ctypes.c_int, _dp]),
            "orc_primal_obj": (_d, [_dp, _dp, _i64, _i64, _dp, _d, _d]),
            "orc_dual_obj": (_d, [_dp, _i64, _dp, _dp, _i64, _d, _d]),
            "orc_kkt_violation": (_d, [_dp, _dp, _i64, _i64, _dp, _d, _d]),
            "orc_default_opts": (None, [ctypes.POINTER(Opts)]),
            "orc_solve": (ctypes.c_int, [_dp, _dp, _i64, _i64, _d, _d, _d, _d, _dp, _dp, ctypes.POINTER(Opts), _dp,
                                         _dp, ctypes.POINTER(Stats), ctypes.POINTER(Trace), _i64, _lp]),
            "orc_aty_fused": (_i64, [_dp, _dp, _i64, _i64, _dp, _dp, _d, _d, _d, _dp, _lp, _dp, _dp, _dp]),
            "orc_dof": (_d, [_dp, _i64, _lp, _i64, _d]),
            "orc_ols": (ctypes.c_int, [_dp, _dp, _i64, _lp, _i64, _dp, _dp]),
            "orc_criteria": (None, [_d, _d, _i64, _i64, _dp, _dp]),
            "orc_model_select": (ctypes.c_int, [_dp, _dp, _i64, _i64, _dp, _d, _dp, _dp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _f64(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(_dp)


def _A(A):
    A = np.ascontiguousarray(A, dtype=np.float64)
    assert A.ndim == 2, "A must be (n, m): column i of the m x n design is A[i]"
    return A, A.shape[1], A.shape[0], A.ctypes.data_as(_dp)


# --- Section 2: penalty, conjugate, prox -------------------------------------

def prox(t, sigma, l1, l2):
    """Eq. (6) left: prox_{σp}(t), elementwise."""
    f = lib().orc_prox
    return np.vectorize(lambda v: f(float(v), sigma, l1, l2), otypes=[np.float64])(t)


def prox_conj(t, sigma, l1, l2):
    """Eq. (6) right: prox_{p*/σ}(t/σ), elementwise, argument t."""
    f = lib().orc_prox_conj
    return np.vectorize(lambda v: f(float(v), sigma, l1, l2), otypes=[np.float64])(t)


def pstar(z, l1, l2):
    """Prop. 1: p*(z)."""
    z, zp = _f64(np.atleast_1d(z))
    return lib().orc_pstar(zp, len(z), l1, l2)


def penalty(x, l1, l2):
    x, xp = _f64(np.atleast_1d(x))
    return lib().orc_penalty(xp, len(x), l1, l2)


def hstar(y, b):
    y, yp = _f64(y)
    b, bp = _f64(b)
    return lib().orc_hstar(yp, bp, len(y))


# --- products and Section 3 ----------------------------------------------------

def aty(A, y):
    A, m, n, Ap = _A(A)
    y, yp = _f64(y)
    w = np.empty(n)
    lib().orc_aty(Ap, m, n, yp, w.ctypes.data_as(_dp))
    return w


def ax(A, x):
    A, m, n, Ap = _A(A)
    x, xp = _f64(x)
    out = np.empty(m)
    lib().orc_ax(Ap, m, n, xp, out.ctypes.data_as(_dp))
    return out


def psi(A, b, x, y, sigma, l1, l2):
    """Prop. 2(1): ψ(y) (including −‖x‖²/(2σ))."""
    A, m, n, Ap = _A(A)
    return lib().orc_psi(Ap, _f64(b)[1], m, n, _f64(x)[1], _f64(y)[1], sigma, l1, l2)


def grad_psi(A, b, x, y, sigma, l1, l2):
    """Eq. (15): ∇ψ(y)."""
    A, m, n, Ap = _A(A)
    g = np.empty(m)
    b, bp = _f64(b)
    x, xp = _f64(x)
    y, yp = _f64(y)
    lib().orc_grad_psi(Ap, bp, m, n, xp, yp, sigma, l1, l2, g.ctypes.data_as(_dp))
    return g


def zbar(A, x, y, sigma, l1, l2):
    """Prop. 2(2): z̄ = prox_{p*/σ}(x/σ − Aᵀy)."""
    A, m, n, Ap = _A(A)
    z = np.empty(n)
    x, xp = _f64(x)
    y, yp = _f64(y)
    lib().orc_zbar(Ap, m, n, xp, yp, sigma, l1, l2, z.ctypes.data_as(_dp))
    return z


def active_set(t, sigma, l1):
    """Eq. (17): J = {i : |t_i| > σλ1} ascending."""
    t, tp = _f64(t)
    J = np.empty(max(len(t), 1), dtype=np.int64)
    r = lib().orc_active_set(tp, len(t), sigma, l1, J.ctypes.data_as(_lp))
    return J[:r].copy()


def newton_direction(A, J, g, kappa, jitter=0.0):
    """Eq. (18)/(19): d solving (I + κ A_J A_Jᵀ) d = −g.  Returns (d, branch).  jitter > 0 scales the
    factored matrix's diagonal by (1 + jitter) (the retry of S:227, reading R36)."""
    A, m, n, Ap = _A(A)
    J = np.ascontiguousarray(J, dtype=np.int64)
    g, gp = _f64(g)
    d = np.empty(m)
    br = lib().orc_newton_direction(Ap, m, J.ctypes.data_as(_lp), len(J), gp, kappa, jitter, d.ctypes.data_as(_dp))
    if br < 0:
        raise FloatingPointError("oracle Cholesky failed")
    return d, br


def cg_direction(A, J, g, kappa, tol=1e-10, maxit=1000):
    """Algorithm 1 step (1) by conjugate gradient, matrix-free V u = u + κA_J(A_Jᵀu),
    d0 = 0, stop at ‖Vd + g‖ ≤ tol‖g‖ (R32).  Returns (d, iterations)."""
    A, m, n, Ap = _A(A)
    J = np.ascontiguousarray(J, dtype=np.int64)
    g, gp = _f64(g)
    d = np.empty(m)
    it = lib().orc_cg_direction(Ap, m, J.ctypes.data_as(_lp), len(J), gp, kappa, tol, maxit, d.ctypes.data_as(_dp))
    return d, it


def chol(M):
    """Textbook Cholesky: returns lower L (column-major semantics on a symmetric M)."""
    M = np.array(M, dtype=np.float64, order="F")
    N = M.shape[0]
    buf = np.ascontiguousarray(M.T.reshape(-1))  # column-major flat
    rc = lib().orc_chol(buf.ctypes.data_as(_dp), N)
    if rc != 0:
        raise FloatingPointError("not SPD")
    L = buf.reshape(N, N).T.copy()
    return np.tril(L)


def primal_obj(A, b, x, l1, l2):
    """Eq. (1)."""
    A, m, n, Ap = _A(A)
    return lib().orc_primal_obj(Ap, _f64(b)[1], m, n, _f64(x)[1], l1, l2)


def dual_obj(b, y, w, l1, l2):
    """−h*(y) − p*(w) with w = Aᵀy (reading R2)."""
    b, bp = _f64(b)
    y, yp = _f64(y)
    w, wp = _f64(w)
    return lib().orc_dual_obj(bp, len(b), yp, wp, len(w), l1, l2)


def kkt_violation(A, b, x, l1, l2):
    """max_i v_i of the KKT inclusion Aᵀ(b−Ax) − λ2x ∈ λ1∂‖x‖₁."""
    A, m, n, Ap = _A(A)
    return lib().orc_kkt_violation(Ap, _f64(b)[1], m, n, _f64(x)[1], l1, l2)


def default_opts(**kw) -> Opts:
    o = Opts()
    lib().orc_default_opts(ctypes.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def solve(A, b, l1, l2, sigma0=5e-3, tol=1e-6, x0=None, trace_cap=0, y0=None, **opts):
    """Algorithm 1 (SsNAL-EN).  y0: the dual start of a warm-started path point (reading R39; None:
    y0 = A x0 − b for a warm start, R8).  Returns (x, y, stats dict, trace list)."""
    A, m, n, Ap = _A(A)
    b, bp = _f64(b)
    o = default_opts(**opts)
    x = np.empty(n)
    y = np.empty(m)
    st = Stats()
    x0p = None
    if x0 is not None:
        x0, x0p = _f64(x0)
    y0p = None
    if y0 is not None:
        y0, y0p = _f64(y0)
    tr = (Trace * max(trace_cap, 1))()
    tl = ctypes.c_int64(0)
    lib().orc_solve(Ap, bp, m, n, l1, l2, sigma0, tol, x0p, y0p, ctypes.byref(o), x.ctypes.data_as(_dp),
                    y.ctypes.data_as(_dp), ctypes.byref(st), tr if trace_cap else None, trace_cap, ctypes.byref(tl))
    stats = {f: getattr(st, f) for f, _ in Stats._fields_}
    stats["branch_steps"] = list(st.branch_steps)
    trace = [{f: getattr(tr[i], f) for f, _ in Trace._fields_} for i in range(min(tl.value, trace_cap))]
    return x, y, stats, trace


def solve_path_lambdas(A, b, ls, sigma0=5e-3, tol=1e-6, x0=None, carry_sigma=True, max_active=None,
                       carry_dual=True, **opts):
    """Warm-started λ path over explicit (λ1, λ2) pairs: point i starts from point i−1's x
    (the warm start of P:411; y0 = A x0 − b by reading R8) and, with carry_sigma, from point i−1's
    final σ — the σ of its last inner solve (reading R38: the paper's "usually SsNAL-EN converges in
    just one iteration", needs the σ the previous point ended with; SPEC's open question S:336
    records the same choice).  With carry_dual (reading R39, P:236-246 + P:409-411: "the solution at the
    previous value" is Algorithm 1's whole starting point) point i > 0 also starts at point i − 1's
    final y instead of y0 = A x0 − b, so no Aᵀ pass is spent on the warm start.  Point 0 starts at
    sigma0 from x0 (None = cold).  The path stops after the first point with at least max_active
    nonzeros.  Returns a list of (x, y, stats)."""
    out = []
    x = x0
    y = None
    sig = sigma0
    for i, (l1, l2) in enumerate(ls):
        x, y, st, _ = solve(A, b, l1, l2, sigma0=sig, tol=tol, x0=x, y0=y if (carry_dual and i > 0) else None,
                            **opts)
        out.append((x, y, st))
        if carry_sigma:
            sig = st["sigma_final"]
        if max_active is not None and st["active"] >= max_active:
            break
    return out


def solve_path(A, b, alpha, cs, sigma0=5e-3, tol=1e-6, carry_sigma=True, max_active=None, carry_dual=True, **opts):
    """The λ path of Section 3.3 on the c grid: λmax = ‖Aᵀb‖∞/α, λ1 = cαλmax, λ2 = c(1−α)λmax
    (P:506), warm-started as in solve_path_lambdas.  Returns (lambdas, [(x, y, stats)])."""
    lm = lambda_max_l1(A, b) / alpha
    ls = [(c * alpha * lm, c * (1 - alpha) * lm) for c in cs]
    res = solve_path_lambdas(A, b, ls, sigma0=sigma0, tol=tol, carry_sigma=carry_sigma, max_active=max_active,
                             carry_dual=carry_dual, **opts)
    return ls[:len(res)], res


def aty_fused(A, b, y, x, sigma, l1, l2, with_grad=True):
    """K1-equivalent: (w, J, P_J, partials[4], g)."""
    A, m, n, Ap = _A(A)
    b, bp = _f64(b)
    y, yp = _f64(y)
    x, xp = _f64(x)
    w = np.empty(n)
    J = np.empty(max(n, 1), dtype=np.int64)
    PJ = np.empty(max(n, 1))
    part = np.empty(4)
    g = np.empty(m) if with_grad else None
    r = lib().orc_aty_fused(Ap, bp, m, n, yp, xp, sigma, l1, l2, w.ctypes.data_as(_dp), J.ctypes.data_as(_lp),
                            PJ.ctypes.data_as(_dp), part.ctypes.data_as(_dp),
                            g.ctypes.data_as(_dp) if with_grad else None)
    return w, J[:r].copy(), PJ[:r].copy(), part, g


def lambda_max_l1(A, b):
    """‖Aᵀb‖∞."""
    return float(np.max(np.abs(aty(A, b))))


# --- Section 3.3: model selection along the path -------------

def dof(A, J, l2):
    """ν = tr(A_J (A_JᵀA_J + λ2 I)⁻¹ A_Jᵀ)."""
    A, m, n, Ap = _A(A)
    J = np.ascontiguousarray(J, dtype=np.int64)
    return lib().orc_dof(Ap, m, J.ctypes.data_as(_lp), len(J), l2)


def ols(A, b, J):
    """De-biased least squares on columns J.  Returns (v, rss, ok)."""
    A, m, n, Ap = _A(A)
    J = np.ascontiguousarray(J, dtype=np.int64)
    b, bp = _f64(b)
    v = np.empty(max(len(J), 1))
    rss = ctypes.c_double(0)
    rc = lib().orc_ols(Ap, bp, m, J.ctypes.data_as(_lp), len(J), v.ctypes.data_as(_dp), ctypes.byref(rss))
    return v[:len(J)].copy(), rss.value, rc == 0


def criteria(rss, nu, m, n):
    """Eq. (21): (gcv, e-bic)."""
    g, e = ctypes.c_double(0), ctypes.c_double(0)
    lib().orc_criteria(rss, nu, m, n, ctypes.byref(g), ctypes.byref(e))
    return g.value, e.value


def model_select(A, b, x, l2):
    """(r, ν, rss, gcv, e-bic, x_debiased) of a solution x."""
    A, m, n, Ap = _A(A)
    b, bp = _f64(b)
    x, xp = _f64(x)
    xdb = np.empty(n)
    out = np.empty(5)
    lib().orc_model_select(Ap, bp, m, n, xp, l2, xdb.ctypes.data_as(_dp), out.ctypes.data_as(_dp))
    return int(out[0]), out[1], out[2], out[3], out[4], xdb


# --- k-fold cross-validation along the λ path (Section 3.3) ----------

def cv_folds(m, k):
    """Fold f holds rows r with r ≡ f (mod k) (reading R35: interleaved, deterministic)."""
    return [np.arange(f, m, k) for f in range(k)]


def residual_ss(A, b, x):
    """‖A x − b‖² by its definition (A is (n, m): row i is column a_i)."""
    r = oracle_ax(A, x) - np.asarray(b, dtype=np.float64)
    return float(r @ r)


def oracle_ax(A, x):
    A, m, n, Ap = _A(A)
    x, xp = _f64(x)
    out = np.empty(m)
    lib().orc_ax(Ap, m, n, xp, out.ctypes.data_as(_dp))
    return out


def cv_path(A, b, alpha, cs, k=5, sigma0=5e-3, tol=1e-6, carry_sigma=True, carry_dual=True):
    """k-fold CV error along c ∈ cs ("cross-validation ... along the path"): λ from the FULL
    data (λmax = ‖Aᵀb‖∞/α) so every fold uses the same grid; for each fold the
    warm-started path on the training rows (σ carried, R38), and the held-out squared error.
    Returns cv[c] = Σ_folds ‖b_test − A_test x_fold(c)‖² / m (reading R35) and the minimising index."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    n, m = A.shape
    lm = float(np.max(np.abs(aty(A, b)))) / alpha
    err = np.zeros(len(cs))
    for test in cv_folds(m, k):
        train = np.setdiff1d(np.arange(m), test)
        Atr, btr = np.ascontiguousarray(A[:, train]), b[train]
        Ate, bte = np.ascontiguousarray(A[:, test]), b[test]
        ls = [(c * alpha * lm, c * (1 - alpha) * lm) for c in cs]
        for i, (x, _, _) in enumerate(solve_path_lambdas(Atr, btr, ls, sigma0=sigma0, tol=tol,
                                                          carry_sigma=carry_sigma, carry_dual=carry_dual)):
            err[i] += residual_ss(Ate, bte, x)
    err /= m
    return err, int(np.argmin(err))
