#!/usr/bin/env python3
"""Phase profile of k_small_solve (build: nvcc -DSMALL_PROF … -o paper_2006_03970_b200/libssnal_en_prof.so).
Prints the thread-0 cycle totals per phase for a cfg1 solve."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import synth  # noqa: E402
import paper_2006_03970_b200.ssnal_en as se  # noqa: E402

se.LIB_PATH = os.path.join(ROOT, "paper_2006_03970_b200", "libssnal_en_prof.so")
lib = se.load_library()
lib.ssnal_en_small_prof.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
cfg = synth.CONFIGS["cfg1"]
A = synth.design(cfg)
b, _ = synth.response(cfg)
variant = int(os.environ.get("SMALL_CLUSTER", "1"))
names = ["pass", "epilogue", "gradient", "gram", "factor", "bwd+d+gd", "-", "-"] if not variant else ["pass", "local-epi", "exchange", "newton-mat", "factor", "bwd+d+gd", "gradient", "panel"]
with se.Problem(A, b) as P:
    P.set_option("small_cluster", variant)
    lm = P.lambda_max_l1 / cfg.alpha
    l1, l2 = 0.5 * cfg.alpha * lm, 0.5 * (1 - cfg.alpha) * lm
    for _ in range(3):
        x, st = P.solve(l1, l2, cfg.sigma0, cfg.tol)
    buf = (ctypes.c_ulonglong * 8)()
    lib.ssnal_en_small_prof(buf, 1)
    reps = 5
    for _ in range(reps):
        x, st = P.solve(l1, l2, cfg.sigma0, cfg.tol)
    lib.ssnal_en_small_prof(buf, 0)
    print("device time per solve (us):", st["time_device_s"] * 1e6, "newton", st["newton_iters"], "outer", st["outer_iters"])
    for k in range(8):
        v = buf[k]
        if k == 6 and variant:  # high half: Σ N of the factorisations (cluster kernel)
            print("sum N per solve:", (v >> 32) / reps)
            v &= 0xFFFFFFFF
        print(f"{names[k]:10s} {v / reps / 1.9e3:8.1f} us per solve")
