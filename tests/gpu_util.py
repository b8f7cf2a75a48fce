"""Helpers for the -m gpu tests: device buffers via torch, parity metrics (BASELINE north star)."""
import numpy as np

try:
    import torch
except Exception:  # pragma: no cover
    torch = None


def cuda_ok():
    return torch is not None and torch.cuda.is_available()


def dev(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def empty(n, dtype=None):
    return torch.empty(max(int(n), 1), dtype=dtype or torch.float64, device="cuda")


def host(t, n=None):
    a = t.cpu().numpy()
    return a if n is None else a[:n]


def aty_errors(w_gpu, w_cpu, A, y):
    """Reading R21: max_i |Δw_i| / (‖a_i‖‖y‖) and ‖Δw‖/‖w‖."""
    colnorm = np.sqrt((A * A).sum(axis=1))
    ny = np.linalg.norm(y)
    d = np.abs(w_gpu - w_cpu)
    e1 = float(np.max(d / (colnorm * ny))) if len(d) else 0.0
    e2 = float(np.linalg.norm(d) / max(np.linalg.norm(w_cpu), 1e-300))
    return e1, e2


def solution_parity(x_gpu, x_cpu, F_gpu, F_cpu):
    """BASELINE north star tolerances: objective 1e-9 rel, ‖Δx‖∞ ≤ 1e-6‖x_cpu‖∞, sign pattern (R22).
    ‖x_cpu‖∞ is floored at R22's 1e-8 (below it a coefficient counts as zero): at λ1 one ulp below
    ‖Aᵀb‖∞ (c = 1 on a grid, R11) the exact solution is O(ulp) and either side may return 0."""
    obj_rel = abs(F_gpu - F_cpu) / max(abs(F_cpu), 1e-300)
    xinf = max(float(np.max(np.abs(x_cpu))) if len(x_cpu) else 0.0, 1e-8)
    dx = float(np.max(np.abs(x_gpu - x_cpu))) if len(x_cpu) else 0.0
    mask = np.maximum(np.abs(x_gpu), np.abs(x_cpu)) > 1e-8
    sign_ok = bool(np.array_equal(np.sign(x_gpu[mask]), np.sign(x_cpu[mask])))
    return {"obj_rel": obj_rel, "xinf_rel": dx / max(xinf, 1e-300), "sign_match": sign_ok,
            "ok": obj_rel <= 1e-9 and dx <= 1e-6 * xinf and sign_ok}


def separated_threshold(t, r_target):
    """A threshold strictly between the r_target-th and (r_target+1)-th largest |t| (no ties)."""
    a = np.sort(np.abs(t))[::-1]
    if r_target <= 0:
        return float(a[0]) * 1.5 + 1.0
    if r_target >= len(a):
        return float(a[-1]) * 0.5
    return float(0.5 * (a[r_target - 1] + a[r_target]))


def compare_to_oracle(A, b, l1, l2, gpu_solve, sigma0=5e-3, tol=1e-6, x0=None, label="", orc_opts=None,
                      rerun_tol=1e-10):
    """Iteration-level parity of one solve ("GPU vs oracle"): both run the same
    iteration, so the outer and Newton counts are expected equal.  A ±1 Newton (or outer) difference —
    a borderline stop or Armijo test at roundoff — triggers a rerun of BOTH at tol = 1e-10, which must
    then meet the BASELINE tolerances; a larger difference fails.  gpu_solve(sigma0, tol, x0) -> (x, stats).
    Checks: solution parity (objective 1e-9 rel, ‖Δx‖∞ ≤ 1e-6‖x_cpu‖∞, sign pattern R22), the GPU's
    primal objective report, the dual objective D(y) = −h*(y) − p*(Aᵀy) at the final y (Prop. 1,
    P:113-125; (D) P:209) and the gap F − D against the oracle's.  Returns (parity dict, stats_gpu,
    stats_cpu, rerun flag)."""
    import oracle

    orc_opts = orc_opts or {}
    xc, yc, stc, _ = oracle.solve(A, b, l1, l2, sigma0=sigma0, tol=tol, x0=x0, **orc_opts)
    xg, stg = gpu_solve(sigma0, tol, x0)
    assert stg["status"] == stc["status"], (label, stg, stc)
    dn = abs(stg["newton_iters"] - stc["newton_iters"])
    do = abs(stg["outer_iters"] - stc["outer_iters"])
    assert dn <= 1 and do <= 1, (label, "iteration counts differ by more than 1", stg, stc)
    rerun = dn + do > 0
    if rerun:
        xc, yc, stc, _ = oracle.solve(A, b, l1, l2, sigma0=sigma0, tol=rerun_tol, x0=x0, **orc_opts)
        xg, stg = gpu_solve(sigma0, rerun_tol, x0)
        assert stg["status"] == stc["status"] == 0, (label, "rerun", stg, stc)
    Fg = oracle.primal_obj(A, b, xg, l1, l2)
    Fc = oracle.primal_obj(A, b, xc, l1, l2)
    par = solution_parity(xg, xc, Fg, Fc)
    assert par["ok"], (label, "rerun" if rerun else "", par, stg, stc)
    assert abs(stg["primal_obj"] - Fg) <= 1e-12 * abs(Fg), (label, stg["primal_obj"], Fg)
    if l2 > 0:
        # D at the final y: the oracle's D(y_cpu) (its stats; equals dual_obj(b, y, Aᵀy)) vs the GPU's D(y_gpu)
        assert stc["dual_obj"] == oracle.dual_obj(b, yc, oracle.aty(A, yc), l1, l2)
        assert abs(stg["dual_obj"] - stc["dual_obj"]) <= 1e-9 * abs(Fc), (label, stg["dual_obj"], stc["dual_obj"])
        assert abs(stg["gap"] - stc["gap"]) <= 1e-9 * abs(Fc), (label, stg["gap"], stc["gap"])
        assert stg["gap"] >= -1e-9 * abs(Fg)
    else:
        assert np.isnan(stg["dual_obj"])
    par.update(rerun=rerun, dual_rel=abs(stg["dual_obj"] - stc["dual_obj"]) / abs(Fc) if l2 > 0 else None)
    return par, stg, stc, rerun
