"""Seeded synthetic inputs shared by the CUDA path and the oracle.

This package holds no SsNAL-EN arithmetic.  It generates the design matrix A
(column-major m x n, i.e. a row-major (n, m) array), the sparse truth x*, and
the response b = A x* + noise for the BASELINE.json configurations, following
the recipe in DESIGN.md ("Input recipe").  The same counter-based generator
(gen_core.h) is compiled for the host (libsynth.so, gcc) and for the device
(libsynth_cuda.so, nvcc), and both produce identical bytes.

Lambda values are NOT produced here: lambda_max = ||A^T b||_inf is method
arithmetic and is computed by the caller (oracle in tests, the C-ABI in bench).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
HOST_LIB = os.path.join(_HERE, "libsynth.so")
DEV_LIB = os.path.join(_HERE, "libsynth_cuda.so")

IID_UNIT_L2, IID_STD, AR1_STD, GENO_STD = 1, 2, 3, 4


@dataclass(frozen=True)
class Config:
    """One BASELINE.json configuration ("Input recipe")."""

    name: str
    m: int
    n: int
    kind: int
    k: int            # nonzeros of x*
    lo: float         # |x*_i| ~ U[lo, hi]
    hi: float
    snr: float
    alpha: float
    cs: tuple         # c values: lambda1 = c*alpha*lmax, lambda2 = c*(1-alpha)*lmax
    seed: int
    path: bool = False  # warm-started path over cs (cfg2)
    sigma0: float = 5e-3
    tol: float = 1e-6
    extra: dict = field(default_factory=dict)


CONFIGS = {
    # BASELINE.json configs[0]: Tiny
    "cfg1": Config("cfg1", 50, 1_000, IID_UNIT_L2, 5, 1.0, 2.0, 5.0, 0.7, (0.5,), 1),
    # configs[1]: Paper-scale simulation, AR(1) Toeplitz 0.5^|i-j|, path c = 0.9..0.1 (R17)
    "cfg2": Config("cfg2", 500, 100_000, AR1_STD, 20, 1.0, 2.0, 5.0, 0.7,
                   tuple(float(c) for c in np.linspace(0.9, 0.1, 10)), 2, path=True),
    # configs[2]: Ultra-high-dim
    "cfg3": Config("cfg3", 500, 1_000_000, IID_STD, 50, 1.0, 2.0, 10.0, 0.5, (0.5, 0.2, 0.05), 3),
    # configs[3]: Genotype-like
    "cfg4": Config("cfg4", 800, 2_000_000, GENO_STD, 30, 0.1, 0.3, 1.0, 0.5, (0.3,), 4),
    # configs[4]: HBM-bound stress
    "cfg5": Config("cfg5", 500, 10_000_000, IID_STD, 100, 1.0, 2.0, 5.0, 0.7, (0.5, 0.1), 5),
}


def scaled(cfg: Config, n: int | None = None, m: int | None = None) -> Config:
    """Same recipe with a different n (and/or m): used for CPU-sized parity cases."""
    from dataclasses import replace

    return replace(cfg, n=n if n is not None else cfg.n, m=m if m is not None else cfg.m)


_host = None
_dev = None


def host_lib():
    global _host
    if _host is None:
        if not os.path.exists(HOST_LIB):
            raise RuntimeError(f"{HOST_LIB} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(HOST_LIB)
        i64, u64, dp, lp = ctypes.c_int64, ctypes.c_uint64, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)
        lib.synth_fill_A.argtypes = [ctypes.c_int, u64, i64, i64, i64, i64, dp]
        lib.synth_fill_A.restype = ctypes.c_int
        lib.synth_columns.argtypes = [ctypes.c_int, u64, i64, i64, lp, i64, dp]
        lib.synth_columns.restype = ctypes.c_int
        lib.synth_xstar.argtypes = [u64, i64, i64, ctypes.c_double, ctypes.c_double, lp, dp]
        lib.synth_xstar.restype = ctypes.c_int
        lib.synth_response.argtypes = [ctypes.c_int, u64, i64, i64, i64, lp, dp, ctypes.c_double, dp, dp]
        lib.synth_response.restype = ctypes.c_int
        lib.synth_normals.argtypes = [u64, u64, i64, dp]
        lib.synth_normals.restype = None
        lib.synth_uniforms.argtypes = [u64, u64, i64, dp]
        lib.synth_uniforms.restype = None
        lib.synth_geno_codes.argtypes = [u64, i64, i64, i64, i64, ctypes.c_void_p, i64, dp]
        lib.synth_geno_codes.restype = ctypes.c_int
        _host = lib
    return _host


def dev_lib():
    global _dev
    if _dev is None:
        if not os.path.exists(DEV_LIB):
            raise RuntimeError(f"{DEV_LIB} missing: run the build")
        lib = ctypes.CDLL(DEV_LIB)
        lib.synth_fill_A_device.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64,
                                            ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        lib.synth_fill_A_device.restype = ctypes.c_int
        lib.synth_geno_codes_device.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                                ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                                ctypes.c_void_p]
        lib.synth_geno_codes_device.restype = ctypes.c_int
        _dev = lib
    return _dev


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _lp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def design(cfg: Config, j0: int = 0, j1: int | None = None) -> np.ndarray:
    """Columns [j0, j1) of A as a C-contiguous (j1-j0, m) float64 array (= column-major m x n)."""
    j1 = cfg.n if j1 is None else j1
    out = np.empty((j1 - j0, cfg.m), dtype=np.float64)
    rc = host_lib().synth_fill_A(cfg.kind, cfg.seed, cfg.m, cfg.n, j0, j1, _dp(out))
    if rc != 0:
        raise RuntimeError(f"synth_fill_A returned {rc}")
    return out


def columns(cfg: Config, idx) -> np.ndarray:
    """Arbitrary standardised columns idx of A, shape (len(idx), m)."""
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    out = np.empty((len(idx), cfg.m), dtype=np.float64)
    rc = host_lib().synth_columns(cfg.kind, cfg.seed, cfg.m, cfg.n, _lp(idx), len(idx), _dp(out))
    if rc != 0:
        raise RuntimeError(f"synth_columns returned {rc}")
    return out


def truth(cfg: Config):
    """(support indices ascending, values) of x*."""
    idx = np.empty(cfg.k, dtype=np.int64)
    val = np.empty(cfg.k, dtype=np.float64)
    rc = host_lib().synth_xstar(cfg.seed, cfg.n, cfg.k, cfg.lo, cfg.hi, _lp(idx), _dp(val))
    if rc != 0:
        raise RuntimeError("synth_xstar failed")
    return idx, val


def response(cfg: Config):
    """b = A x* + eps (regenerates only the support columns).  Returns (b, noise_sd)."""
    idx, val = truth(cfg)
    b = np.empty(cfg.m, dtype=np.float64)
    sd = np.zeros(1, dtype=np.float64)
    rc = host_lib().synth_response(cfg.kind, cfg.seed, cfg.m, cfg.n, cfg.k, _lp(idx), _dp(val), cfg.snr,
                                   _dp(b), _dp(sd))
    if rc != 0:
        raise RuntimeError(f"synth_response returned {rc}")
    return b, float(sd[0])


def normals(seed: int, sub: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.float64)
    host_lib().synth_normals(seed, sub, count, _dp(out))
    return out


def uniforms(seed: int, sub: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.float64)
    host_lib().synth_uniforms(seed, sub, count, _dp(out))
    return out


def fill_device(cfg: Config, dptr: int, stream: int = 0, j0: int = 0, j1: int | None = None) -> None:
    """Write columns [j0, j1) of A into device memory at dptr (column-major, lda = m)."""
    j1 = cfg.n if j1 is None else j1
    rc = dev_lib().synth_fill_A_device(cfg.kind, cfg.seed, cfg.m, cfg.n, j0, j1, ctypes.c_void_p(dptr),
                                       ctypes.c_void_p(stream))
    if rc != 0:
        raise RuntimeError(f"synth_fill_A_device returned {rc}")


def geno_stride(m: int) -> int:
    """Bytes per packed genotype column: ceil(m/4) rounded up to 16 (TMA-aligned tiles)."""
    return ((m + 3) // 4 + 15) // 16 * 16


def geno_codes(cfg: Config, j0: int = 0, j1: int | None = None):
    """Compressed storage of a GENO_STD design: (codes uint8 (ncols, stride), tab (ncols, 3)).
    decode_geno(codes, tab, m) equals design(cfg) bit for bit."""
    assert cfg.kind == GENO_STD
    j1 = cfg.n if j1 is None else j1
    stride = geno_stride(cfg.m)
    codes = np.empty((j1 - j0, stride), dtype=np.uint8)
    tab = np.empty((j1 - j0, 3), dtype=np.float64)
    rc = host_lib().synth_geno_codes(cfg.seed, cfg.m, cfg.n, j0, j1, codes.ctypes.data, stride, _dp(tab))
    if rc < 0:
        raise RuntimeError(f"synth_geno_codes returned {rc}")
    return codes, tab


def decode_geno(codes: np.ndarray, tab: np.ndarray, m: int) -> np.ndarray:
    """(ncols, m) fp64 design from packed codes: entry (j, k) = tab[j, (codes[j, k//4] >> 2(k%4)) & 3]."""
    k = np.arange(m)
    g = (codes[:, k // 4] >> (2 * (k % 4))) & 3
    return np.take_along_axis(tab, g.astype(np.int64), axis=1)


def fill_device_geno(cfg: Config, dcodes: int, dtab: int, stream: int = 0, j0: int = 0, j1: int | None = None):
    """Device twin of geno_codes: packed codes (stride geno_stride(m)) and tables into device memory."""
    j1 = cfg.n if j1 is None else j1
    rc = dev_lib().synth_geno_codes_device(cfg.seed, cfg.m, cfg.n, j0, j1, ctypes.c_void_p(dcodes),
                                           geno_stride(cfg.m), ctypes.c_void_p(dtab), ctypes.c_void_p(stream))
    if rc < 0:
        raise RuntimeError(f"synth_geno_codes_device returned {rc}")
