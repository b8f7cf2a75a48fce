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
    """BASELINE north star tolerances: objective 1e-9 rel, ‖Δx‖∞ ≤ 1e-6‖x_cpu‖∞, sign pattern (R22)."""
    obj_rel = abs(F_gpu - F_cpu) / max(abs(F_cpu), 1e-300)
    xinf = float(np.max(np.abs(x_cpu))) if len(x_cpu) else 0.0
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
