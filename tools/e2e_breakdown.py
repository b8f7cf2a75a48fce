#!/usr/bin/env python3
"""Wall-clock split of the host-memory C-ABI calls (create from pinned host buffers / the solves / destroy) on a
BASELINE config: where the e2e number of bench.py goes.  Usage: tools/e2e_breakdown.py cfg2 [reps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2006_03970_b200 import Problem  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = synth.CONFIGS[name]
A = torch.empty((cfg.n, cfg.m), dtype=torch.float64, pin_memory=True)
A.copy_(torch.from_numpy(synth.design(cfg)))
b, _ = synth.response(cfg)
An = A.numpy()
for it in range(reps + 1):
    t0 = time.perf_counter()
    P = Problem(An, b)
    t1 = time.perf_counter()
    lm = P.lambda_max_l1 / cfg.alpha
    x = None
    for c in cfg.cs:
        x, st = P.solve(c * cfg.alpha * lm, c * (1 - cfg.alpha) * lm, cfg.sigma0, cfg.tol, x0=x if cfg.path else None)
    t2 = time.perf_counter()
    P.close()
    t3 = time.perf_counter()
    if it:
        print(f"{name}: create {1e3 * (t1 - t0):.3f} ms (H2D floor at 55 GB/s: {8e3 * cfg.m * cfg.n / 55e9:.3f} ms)  "
              f"solves {1e3 * (t2 - t1):.3f} ms  destroy {1e3 * (t3 - t2):.3f} ms", flush=True)
