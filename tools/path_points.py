#!/usr/bin/env python3
"""Per-point device time of the cfg2 warm-started path (ssnal_en_solve_path_device, σ and the dual
iterate carried): how much of a point is fixed overhead (init, objective, copies, graph launch)
versus Newton steps.  Prints one line per point: c, outer, Newton, A passes, device µs."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2006_03970_b200 import Problem  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
m, n = cfg.m, cfg.n
st = torch.cuda.current_stream()
dA = torch.empty((n, m), dtype=torch.float64, device="cuda")
synth.fill_device(cfg, dA.data_ptr(), st.cuda_stream)
b, _ = synth.response(cfg)
db = torch.from_numpy(b).cuda()
P = Problem.from_device(dA.data_ptr(), db.data_ptr(), m, n, st.cuda_stream, keep=(dA, db))
lm = P.lambda_max_l1 / cfg.alpha
l1s = [c * cfg.alpha * lm for c in cfg.cs]
l2s = [c * (1 - cfg.alpha) * lm for c in cfg.cs]
X = torch.zeros((len(cfg.cs), n), dtype=torch.float64, device="cuda")
for _ in range(3):
    P.solve_path_device(l1s, l2s, cfg.sigma0, cfg.tol, 0, X.data_ptr())
sts = P.solve_path_device(l1s, l2s, cfg.sigma0, cfg.tol, 0, X.data_ptr())
tot = 0.0
for c, s in zip(cfg.cs, sts):
    tot += s["time_device_s"]
    print(f"c={c:.3f} outer={s['outer_iters']} newton={s['newton_iters']} passes={s['aty_passes']} "
          f"backtracks={s['backtracks']} launches={s['kernel_launches']} device={s['time_device_s'] * 1e6:8.1f} us")
print(f"total {tot * 1e3:.3f} ms")
