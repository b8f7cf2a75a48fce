#!/usr/bin/env python3
"""One Newton-direction call (K3 Gram + reduce, K4 cluster Cholesky, SMW back-substitution) at a
chosen active-set size r, m = 500 iid design — the target for `ncu -k regex:'k_gram|k_chol|k_smw'`.

  python tools/ncu_newton.py --r 1165      # m × m branch (cfg3 c = 0.05 size)
  python tools/ncu_newton.py --r 435       # SMW branch (cfg2 c = 0.1 size)
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2006_03970_b200 import Problem  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--r", type=int, default=1165)
    ap.add_argument("--m", type=int, default=500)
    ap.add_argument("--n", type=int, default=20000)
    ap.add_argument("--kappa", type=float, default=0.01)
    ap.add_argument("--calls", type=int, default=1)
    args = ap.parse_args()
    m, n, r = args.m, args.n, args.r
    cfg = synth.Config("t", m, n, synth.IID_STD, 5, 1.0, 2.0, 5.0, 0.7, (0.5,), 3)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    with Problem(A, b) as P:
        g = torch.from_numpy(synth.normals(3, 8, m)).cuda()
        d = torch.empty(m, dtype=torch.float64, device="cuda")
        J = torch.from_numpy(np.sort(np.argsort(synth.uniforms(3, 7, n))[:r]).astype(np.int32)).cuda()
        for _ in range(args.calls):
            gd, br = P.newton_direction(J.data_ptr(), r, g.data_ptr(), args.kappa, d.data_ptr())
        torch.cuda.synchronize()
        print(f"m={m} r={r} branch={br} gd={gd:.6e}")


if __name__ == "__main__":
    main()
