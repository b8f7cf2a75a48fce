#!/usr/bin/env python3
"""Per-Newton-step trace of the oracle on a BASELINE config (branch, r = |J|, step length, res1),
for deciding where the Newton-system kernels (K3/K4) spend their time.  Test infrastructure use
of the oracle only (no product code).  Usage: tools/trace_steps.py cfg5 [c ...]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402

name = sys.argv[1]
cfg = synth.CONFIGS[name]
cs = [float(v) for v in sys.argv[2:]] or list(cfg.cs)
A = synth.design(cfg)
b, _ = synth.response(cfg)
lm = oracle.lambda_max_l1(A, b) / cfg.alpha
x, sig = None, cfg.sigma0
for c in cs:
    l1, l2 = c * cfg.alpha * lm, c * (1 - cfg.alpha) * lm
    x0 = x if cfg.path else None
    xs, _, st, tr = oracle.solve(A, b, l1, l2, sigma0=sig if cfg.path else cfg.sigma0, tol=cfg.tol, x0=x0,
                                 trace_cap=200)
    if cfg.path:
        x, sig = xs, st["sigma_final"]
    print(json.dumps({"cfg": name, "c": c, "outer": st["outer_iters"], "newton": st["newton_iters"],
                      "steps": [(t["outer"], t["branch"], t["r"], t["s"]) for t in tr]}), flush=True)
