"""ctypes binding of include/ssnal_en.h (argument marshalling only).

Names follow the C ABI: ssnal_en_create / _create_device / _solve / _solve_device /
_aty_fused / _epilogue / _newton_direction / _lambda_max_l1 / _set_option /
_get_info / _destroy.  Device pointers are passed as integers (e.g.
torch.Tensor.data_ptr()); host arrays as numpy float64 arrays.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libssnal_en.so")

SSNAL_OK, SSNAL_NOT_CONVERGED, SSNAL_EINVAL, SSNAL_ECUDA, SSNAL_ENUMERIC = 0, 1, 2, 3, 4

_d = ctypes.c_double
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_vp = ctypes.c_void_p
_dp = ctypes.POINTER(ctypes.c_double)


class Stats(ctypes.Structure):
    """Mirror of ssnal_en_stats."""

    _fields_ = [("status", _i32), ("outer_iters", _i32), ("newton_iters", _i32), ("psi_evals", _i32),
                ("backtracks", _i32), ("aty_passes", _i32), ("branch_steps", _i32 * 4),
                ("line_search_stalled", _i32), ("cg_iters", _i32), ("active", _i64), ("res_kkt1", _d), ("res_kkt3", _d),
                ("primal_obj", _d), ("dual_obj", _d), ("gap", _d), ("sigma_final", _d),
                ("time_device_s", _d), ("time_total_s", _d), ("kernel_launches", _i64), ("k1_time_s", _d),
                ("k1_launches", _i32), ("jitter_retries", _i32), ("primal_viol", _d)]

    def as_dict(self):
        d = {f: getattr(self, f) for f, _ in self._fields_ if f != "reserved"}
        d["branch_steps"] = list(self.branch_steps)
        return d


class Criteria(ctypes.Structure):
    """Mirror of ssnal_en_criteria."""

    _fields_ = [("active", _i64), ("nu", _d), ("rss", _d), ("gcv", _d), ("ebic", _d), ("ols_ok", _i32),
                ("reserved", _i32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_ if f != "reserved"}


class SsnalError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"ssnal_en error {code}: {msg}")
        self.code = code


_lib = None

# int (*)(void* ctx, double* buf, int64_t count, int op, void* stream) — ssnal_en_allreduce_fn
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                                ctypes.c_void_p)


def load_library():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python tools/build.py` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.POINTER
        L.ssnal_en_create.argtypes = [_dp, _dp, _i64, _i64, P(_vp)]
        L.ssnal_en_create_device.argtypes = [_vp, _vp, _i64, _i64, _vp, P(_vp)]
        L.ssnal_en_create_geno.argtypes = [_vp, _i64, _dp, _dp, _i64, _i64, P(_vp)]
        L.ssnal_en_create_geno_device.argtypes = [_vp, _i64, _vp, _vp, _i64, _i64, _vp, P(_vp)]
        L.ssnal_en_lambda_max_l1.argtypes = [_vp]
        L.ssnal_en_lambda_max_l1.restype = _d
        L.ssnal_en_set_option.argtypes = [_vp, ctypes.c_char_p, _d]
        L.ssnal_en_get_info.argtypes = [_vp, ctypes.c_char_p]
        L.ssnal_en_get_info.restype = _d
        L.ssnal_en_solve.argtypes = [_vp, _d, _d, _d, _d, _dp, _dp, P(Stats)]
        L.ssnal_en_solve_device.argtypes = [_vp, _d, _d, _d, _d, _vp, _vp, P(Stats)]
        L.ssnal_en_solve_path_device.argtypes = [_vp, ctypes.c_int64, _dp, _dp, _d, _d, _vp, _vp, P(Stats)]
        L.ssnal_en_aty_fused.argtypes = [_vp, _vp, _vp, _d, _d, _d, _vp, _vp, _vp, P(_i64), _dp, _vp]
        L.ssnal_en_epilogue.argtypes = [_vp, _vp, _vp, _d, _vp, _d, _d, _d, _vp, _vp, _vp, P(_i64), _dp]
        L.ssnal_en_newton_direction.argtypes = [_vp, _vp, _i64, _vp, _d, _vp, _dp, P(_i32)]
        L.ssnal_en_model_select.argtypes = [_vp, _d, _dp, P(Criteria)]
        L.ssnal_en_model_select.restype = ctypes.c_int
        L.ssnal_en_residual.argtypes = [_vp, _dp, _dp]
        L.ssnal_en_residual_device.argtypes = [_vp, _vp, _dp]
        L.ssnal_en_set_comm.argtypes = [_vp, ALLREDUCE_FN, _vp, ctypes.c_int, ctypes.c_int]
        L.ssnal_en_peer_export.argtypes = [_vp, ctypes.c_int, _vp]
        L.ssnal_en_peer_attach.argtypes = [_vp, ctypes.c_int, ctypes.c_int, _vp]
        L.ssnal_en_peer_selftest.argtypes = [ctypes.c_int, ctypes.c_int, _i64, P(_i64), _dp, _dp]
        L.ssnal_en_destroy.argtypes = [_vp]
        L.ssnal_en_destroy.restype = None
        L.ssnal_en_last_error.restype = ctypes.c_char_p
        L.ssnal_en_version.restype = ctypes.c_char_p
        for f in ("create", "create_device", "create_geno", "create_geno_device", "residual", "residual_device",
                  "set_option", "solve", "solve_device", "aty_fused", "epilogue",
                  "newton_direction", "set_comm", "peer_export", "peer_attach", "peer_selftest"):
            getattr(L, "ssnal_en_" + f).restype = ctypes.c_int
        _lib = L
    return _lib


IPC_HANDLE_BYTES = 64  # SSNAL_EN_IPC_HANDLE_BYTES


def peer_selftest(nranks: int, iters: int, count: int):
    """The exchange protocol of peer-attached sharded solves with nranks ranks emulated as the CTAs of
    one cooperative launch on the current device (ssnal_en_peer_selftest): returns (mismatches,
    last small sums, last big sums) with the sums as (nranks, count) arrays."""
    L = load_library()
    mis = _i64(0)
    small = np.zeros((nranks, count))
    big = np.zeros((nranks, count))
    _check(L.ssnal_en_peer_selftest(nranks, iters, count, ctypes.byref(mis),
                                    small.ctypes.data_as(_dp), big.ctypes.data_as(_dp)))
    return mis.value, small, big


def _check(rc, allow=(SSNAL_OK,)):
    if rc not in allow:
        raise SsnalError(rc, load_library().ssnal_en_last_error().decode())
    return rc


def _f64(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(_dp)


class Problem:
    """Handle around ssnal_en_problem.

    Problem(A, b)                          host arrays; A is (n, m) C-contiguous = column-major m x n
    Problem.from_device(dA, db, m, n, s)   device pointers (borrowed), s = cudaStream_t as int
    Problem.from_geno(codes, tab, b)       packed 2-bit genotype codes (n, stride) uint8 + tables (n, 3)
    Problem.from_geno_device(dcodes, stride, dtab, db, m, n, s)   the same, device pointers (borrowed)
    """

    def __init__(self, A=None, b=None, _handle=None, _keep=None):
        self._lib = load_library()
        self._keep = _keep
        if _handle is not None:
            self._h = _handle
        else:
            A, Ap = _f64(A)
            b, bp = _f64(b)
            n, m = A.shape
            h = _vp()
            _check(self._lib.ssnal_en_create(Ap, bp, m, n, ctypes.byref(h)))
            self._h = h
        self.m = int(self.info("m"))
        self.n = int(self.info("n"))

    @classmethod
    def from_device(cls, dA: int, db: int, m: int, n: int, stream: int = 0, keep=None):
        lib = load_library()
        h = _vp()
        _check(lib.ssnal_en_create_device(_vp(dA), _vp(db), m, n, _vp(stream), ctypes.byref(h)))
        return cls(_handle=h, _keep=keep)

    @classmethod
    def from_geno(cls, codes, tab, b):
        """Compressed genotype storage: a_kj = tab[j, (codes[j, k//4] >> 2(k%4)) & 3]."""
        lib = load_library()
        codes = np.ascontiguousarray(codes, dtype=np.uint8)
        tab, tp = _f64(tab)
        b, bp = _f64(b)
        n, stride = codes.shape
        h = _vp()
        _check(lib.ssnal_en_create_geno(_vp(codes.ctypes.data), stride, tp, bp, len(b), n, ctypes.byref(h)))
        return cls(_handle=h)

    @classmethod
    def from_geno_device(cls, dcodes: int, stride: int, dtab: int, db: int, m: int, n: int, stream: int = 0,
                         keep=None):
        lib = load_library()
        h = _vp()
        _check(lib.ssnal_en_create_geno_device(_vp(dcodes), stride, _vp(dtab), _vp(db), m, n, _vp(stream),
                                               ctypes.byref(h)))
        return cls(_handle=h, _keep=keep)

    # -- introspection / options --
    @property
    def lambda_max_l1(self) -> float:
        return self._lib.ssnal_en_lambda_max_l1(self._h)

    def info(self, key: str) -> float:
        return self._lib.ssnal_en_get_info(self._h, key.encode())

    def set_option(self, key: str, value: float):
        _check(self._lib.ssnal_en_set_option(self._h, key.encode(), float(value)))

    # -- solves --
    def solve(self, lambda1, lambda2, sigma0=5e-3, tol=1e-6, x0=None):
        """Host-memory solve: returns (x, stats dict)."""
        x = np.empty(self.n)
        st = Stats()
        x0p = None
        if x0 is not None:
            x0, x0p = _f64(x0)
        rc = self._lib.ssnal_en_solve(self._h, lambda1, lambda2, sigma0, tol, x0p, x.ctypes.data_as(_dp),
                                      ctypes.byref(st))
        _check(rc, (SSNAL_OK, SSNAL_NOT_CONVERGED, SSNAL_ENUMERIC))
        return x, st.as_dict()

    def residual(self, x) -> float:
        """‖A x − b‖² for this handle's A, b and a host x (cross-validation test folds)."""
        x, xp = _f64(x)
        out = ctypes.c_double(0.0)
        _check(self._lib.ssnal_en_residual(self._h, xp, ctypes.byref(out)))
        return out.value

    def residual_device(self, x_ptr: int) -> float:
        out = ctypes.c_double(0.0)
        _check(self._lib.ssnal_en_residual_device(self._h, _vp(x_ptr), ctypes.byref(out)))
        return out.value

    def solve_device(self, lambda1, lambda2, sigma0, tol, x0_ptr, x_out_ptr):
        st = Stats()
        rc = self._lib.ssnal_en_solve_device(self._h, lambda1, lambda2, sigma0, tol,
                                             _vp(x0_ptr) if x0_ptr else None, _vp(x_out_ptr), ctypes.byref(st))
        _check(rc, (SSNAL_OK, SSNAL_NOT_CONVERGED, SSNAL_ENUMERIC))
        return st.as_dict()

    def solve_path_device(self, lambda1s, lambda2s, sigma0, tol, x0_ptr, x_out_ptr):
        """Warm-started λ path on device buffers (x_out: npts × n); returns the per-point stats dicts."""
        k = len(lambda1s)
        l1 = np.ascontiguousarray(lambda1s, dtype=np.float64)
        l2 = np.ascontiguousarray(lambda2s, dtype=np.float64)
        st = (Stats * k)()
        rc = self._lib.ssnal_en_solve_path_device(self._h, k, l1.ctypes.data_as(_dp), l2.ctypes.data_as(_dp),
                                                  sigma0, tol, _vp(x0_ptr) if x0_ptr else None, _vp(x_out_ptr), st)
        _check(rc, (SSNAL_OK, SSNAL_NOT_CONVERGED, SSNAL_ENUMERIC))
        return [s.as_dict() for s in st]

    def model_select(self, lambda2, debias=False):
        """ν, rss (after OLS de-biasing), GCV, e-BIC of the latest solution.
        Returns (criteria dict, de-biased x or None)."""
        c = Criteria()
        xdb = np.empty(self.n) if debias else None
        rc = self._lib.ssnal_en_model_select(self._h, lambda2, xdb.ctypes.data_as(_dp) if debias else None,
                                             ctypes.byref(c))
        _check(rc)
        return c.as_dict(), xdb

    # -- kernel hooks (device pointers) --
    def aty_fused(self, y, x, sigma, l1, l2, w_out, J_out, PJ_out, grad_out=0):
        r = _i64(0)
        part = (ctypes.c_double * 4)()
        _check(self._lib.ssnal_en_aty_fused(self._h, _vp(y), _vp(x), sigma, l1, l2, _vp(w_out), _vp(J_out),
                                            _vp(PJ_out), ctypes.byref(r), part, _vp(grad_out) if grad_out else None))
        return r.value, list(part)

    def epilogue(self, w0, w1, s, x, sigma, l1, l2, w_out, J_out, PJ_out):
        r = _i64(0)
        part = (ctypes.c_double * 4)()
        _check(self._lib.ssnal_en_epilogue(self._h, _vp(w0), _vp(w1) if w1 else None, s, _vp(x), sigma, l1, l2,
                                           _vp(w_out) if w_out else None, _vp(J_out), _vp(PJ_out),
                                           ctypes.byref(r), part))
        return r.value, list(part)

    def newton_direction(self, J, r, g, kappa, d_out):
        gd = _d(0)
        br = _i32(0)
        _check(self._lib.ssnal_en_newton_direction(self._h, _vp(J) if J else None, r, _vp(g), kappa, _vp(d_out),
                                                   ctypes.byref(gd), ctypes.byref(br)))
        return gd.value, br.value

    def set_comm(self, fn, rank: int, nranks: int):
        """Make this handle rank `rank` of a column-sharded solve (§8(f3)); fn(buf_ptr, count, op,
        stream) -> None all-reduces `count` doubles at the device pointer in place (op 0 sum, 1 max),
        stream-ordered.  See ssnal_en_set_comm in include/ssnal_en.h."""

        def cb(ctx, buf, count, op, stream):
            try:
                fn(buf, count, op, stream)
                return 0
            except Exception:  # reported as SSNAL_ECUDA by the library
                import traceback
                traceback.print_exc()
                return 1

        self._comm_cb = ALLREDUCE_FN(cb)  # kept alive with the handle
        _check(self._lib.ssnal_en_set_comm(self._h, self._comm_cb, None, rank, nranks))

    def peer_export(self, nranks: int) -> bytes:
        """Allocate this rank's exchange region for a peer-memory sharded solve (§8(f3)) and return its
        IPC handle (IPC_HANDLE_BYTES bytes).  See ssnal_en_peer_export in include/ssnal_en.h."""
        buf = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
        _check(self._lib.ssnal_en_peer_export(self._h, nranks, buf))
        return buf.raw

    def peer_attach(self, rank: int, nranks: int, handles):
        """Map the peers' exchange regions (handles: every rank's peer_export bytes, rank order) and
        make this handle rank `rank` of a sharded solve with device-resident exchanges (a collective
        call).  See ssnal_en_peer_attach in include/ssnal_en.h."""
        blob = b"".join(bytes(h) for h in handles)
        if len(handles) != nranks or len(blob) != nranks * IPC_HANDLE_BYTES:
            raise ValueError("need one IPC handle per rank")
        buf = ctypes.create_string_buffer(blob, len(blob))
        _check(self._lib.ssnal_en_peer_attach(self._h, rank, nranks, buf))

    def close(self):
        if getattr(self, "_h", None):
            self._lib.ssnal_en_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
