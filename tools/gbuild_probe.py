import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, numpy as np, synth, torch
from paper_2006_03970_b200 import Problem
cfg = synth.CONFIGS["cfg2"]
A = synth.design(cfg); b, _ = synth.response(cfg)
Ah = torch.from_numpy(A).pin_memory().numpy()
for rep in range(3):
    t0 = time.perf_counter(); P = Problem(Ah, b); t1 = time.perf_counter()
    lm = P.lambda_max_l1 / cfg.alpha
    ts = []
    for i in range(3):
        t = time.perf_counter(); P.solve(0.5 * cfg.alpha * lm, 0.5 * (1 - cfg.alpha) * lm); ts.append(time.perf_counter() - t)
    t2 = time.perf_counter(); P.close(); t3 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} ms, solves {[round(1e3*x,2) for x in ts]} ms, close {1e3*(t3-t2):.1f} ms")
