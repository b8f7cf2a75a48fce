#!/usr/bin/env python3
"""K4 DSMEM-resident vs cluster kernel: the Newton direction through the C ABI for several (m, r),
chol_dsm = 1 vs 0 (max relative difference), plus per-call timing of both."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2006_03970_b200 import Problem  # noqa: E402

cases = [(500, r) for r in (1, 31, 32, 33, 64, 65, 96, 97, 128, 129, 160, 192, 256)] + [(64, 40), (96, 200), (128, 300), (160, 400)]
for m, r in cases:
    n = max(2 * r, 2000)
    cfg = synth.Config("t", m, n, synth.IID_STD, 5, 1.0, 2.0, 5.0, 0.7, (0.5,), 3)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    with Problem(A, b) as P:
        g = torch.from_numpy(synth.normals(3, 8, m)).cuda()
        J = torch.from_numpy(np.sort(np.argsort(synth.uniforms(3, 7, n))[:r]).astype(np.int32)).cuda()
        res = {}
        for dsm in (0, 1):
            P.set_option("chol_dsm", dsm)
            d = torch.empty(m, dtype=torch.float64, device="cuda")
            for _ in range(2):
                gd, br = P.newton_direction(J.data_ptr(), r, g.data_ptr(), 0.01, d.data_ptr())
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(10):
                P.newton_direction(J.data_ptr(), r, g.data_ptr(), 0.01, d.data_ptr())
            torch.cuda.synchronize()
            res[dsm] = (d.cpu().numpy(), gd, br, (time.perf_counter() - t0) / 10 * 1e6)
        d0, d1 = res[0][0], res[1][0]
        err = np.max(np.abs(d1 - d0)) / np.max(np.abs(d0))
        print(f"m={m} r={r} br={res[1][2]} dsm_on={P.info('chol_dsm')} rel={err:.2e} gd {res[0][1]:.6e} {res[1][1]:.6e} "
              f"wall us: old {res[0][3]:.1f} dsm {res[1][3]:.1f}", flush=True)
