#!/usr/bin/env python3
"""Per-kernel device time of one workload step under torch.profiler (CUPTI), warm caches.

  python tools/kprof.py [--config cfg2] [--reps 1]

Prints a table of kernel name, launches, total and mean device time, and the host-side
wall time of the step (the difference is launch / synchronisation overhead).
"""
import argparse
import collections
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import synth  # noqa: E402
import paper_2006_03970_b200.ssnal_en as _se  # noqa: E402

if os.environ.get("SSNAL_EN_LIB"):  # A/B a variant build of the library (probe use only)
    _se.LIB_PATH = os.environ["SSNAL_EN_LIB"]
from paper_2006_03970_b200 import Problem  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--control", default="graph", choices=["graph", "host"])
    ap.add_argument("--newton", default="", help="comma list of r: time the Newton direction hook (m=500)")
    ap.add_argument("--set", action="append", default=[], help="library option key=value (repeatable)")
    args = ap.parse_args()
    if args.newton:
        return newton(args)
    cfg = synth.CONFIGS[args.config]
    if args.n:
        cfg = synth.scaled(cfg, n=args.n)
    m, n = cfg.m, cfg.n
    st = torch.cuda.current_stream()
    dA = torch.empty((n, m), dtype=torch.float64, device="cuda")
    synth.fill_device(cfg, dA.data_ptr(), st.cuda_stream)
    b, _ = synth.response(cfg)
    db = torch.from_numpy(b).cuda()
    P = Problem.from_device(dA.data_ptr(), db.data_ptr(), m, n, st.cuda_stream, keep=(dA, db))
    P.set_option("graph", 1 if args.control == "graph" else 0)
    for kv in args.set:
        k, v = kv.split("=")
        P.set_option(k, float(v))
    lm = P.lambda_max_l1 / cfg.alpha
    x = torch.zeros(n, dtype=torch.float64, device="cuda")

    X = torch.zeros((len(cfg.cs), n), dtype=torch.float64, device="cuda")

    def step():
        if cfg.path:  # the bench's warm-started path (σ carried, one synchronisation per path)
            P.solve_path_device([c * cfg.alpha * lm for c in cfg.cs], [c * (1 - cfg.alpha) * lm for c in cfg.cs],
                                cfg.sigma0, cfg.tol, 0, X.data_ptr())
            return
        for i, c in enumerate(cfg.cs):
            P.solve_device(c * cfg.alpha * lm, c * (1 - cfg.alpha) * lm, cfg.sigma0, cfg.tol, 0, x.data_ptr())

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        t0 = time.perf_counter()
        for _ in range(args.reps):
            step()
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / args.reps
    agg = collections.defaultdict(lambda: [0, 0.0])
    for e in prof.events():
        if e.device_type.name == "CUDA" and e.name:
            k = e.name.split("(")[0][:48]
            agg[k][0] += 1
            agg[k][1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
    tot = sum(v[1] for v in agg.values())
    print(f"wall per step {wall * 1e3:.2f} ms; kernel time per step {tot / 1e3 / args.reps:.2f} ms")
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:40]:
        print(f"{k:48s} {c // args.reps:6d} {t / 1e3 / args.reps:8.3f} ms  {100 * t / tot:5.1f}%  avg {t / c:8.2f} us")


def newton(args):
    import numpy as np

    m = 500
    n = max(4000, 2 * max(int(v) for v in args.newton.split(",")))
    cfg = synth.Config("t", m, n, synth.IID_STD, 5, 1.0, 2.0, 5.0, 0.7, (0.5,), 3)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    P = Problem(A, b)
    for kv in args.set:
        k, v = kv.split("=")
        P.set_option(k, float(v))
    g = torch.from_numpy(synth.normals(3, 8, m)).cuda()
    d = torch.empty(m, dtype=torch.float64, device="cuda")
    for r in [int(v) for v in args.newton.split(",")]:
        J = torch.from_numpy(np.sort(np.argsort(synth.uniforms(3, 7, n))[:r]).astype(np.int32)).cuda()
        for _ in range(3):
            P.newton_direction(J.data_ptr(), r, g.data_ptr(), 0.01, d.data_ptr())
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            t0 = time.perf_counter()
            for _ in range(10):
                P.newton_direction(J.data_ptr(), r, g.data_ptr(), 0.01, d.data_ptr())
            wall = (time.perf_counter() - t0) / 10
        agg = collections.defaultdict(lambda: [0, 0.0])
        for e in prof.events():
            if e.device_type.name == "CUDA" and e.name:
                k = e.name.split("(")[0][:30]
                agg[k][0] += 1
                agg[k][1] += e.device_time_total
        parts = ", ".join(f"{k.split('::')[-1]}={t / c:.1f}" for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]))
        print(f"r={r:5d} wall={wall * 1e6:8.1f} us  kernels(us): {parts}")


if __name__ == "__main__":
    main()
