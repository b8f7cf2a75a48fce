"""Randomised end-to-end parity sweep: seeded random (recipe, m, n, α, c, σ0) problems, each solved on
every execution path of the library — the one-cluster launch (when eligible), the multi-kernel graph,
host-driven control, and the graph with the Aᵀb reuse of reading R40 forced on (no size gate, both of
its modes) — and each compared with the oracle by the SURVEY §8(c) rule (equal counts or the ±1 rerun
of both at tol 1e-10; objective 1e-9, ‖Δx‖∞ ≤ 1e-6‖x‖∞, sign pattern; dual objective and gap).  The
warm-started solve from the cold solution follows on both control modes.  The fixed-shape tests pin the tile edges; this one looks for anything the hand-picked shapes miss."""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import compare_to_oracle, cuda_ok

pytestmark = pytest.mark.gpu

if cuda_ok():
    from paper_2006_03970_b200 import Problem

KINDS = [synth.IID_STD, synth.IID_UNIT_L2, synth.AR1_STD]


def cases(count, seed):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(count):
        m = int(rng.choice([2, 5, 17, 31, 32, 33, 50, 64, 65, 100, 129, 257, 500, 513, 800, 1024]))
        n = int(rng.integers(max(m // 2, 1), 6000))
        if i % 5 == 0:
            n = int(rng.integers(1, 1025))  # the one-cluster path's range
        out.append((KINDS[int(rng.integers(len(KINDS)))], m, n, float(rng.choice([0.9, 0.5, 0.2, 0.05, 0.01])),
                    float(rng.choice([0.3, 0.5, 0.7, 1.0])), float(rng.choice([5e-3, 1e-2, 1.0])),
                    int(rng.integers(1, 10_000))))
    return out


@pytest.mark.parametrize("case", cases(60, 20260321), ids=lambda c: f"k{c[0]}_m{c[1]}_n{c[2]}_c{c[3]}_a{c[4]}_s{c[5]}")
def test_random_problem_all_paths(case):
    kind, m, n, c, alpha, sigma0, seed = case
    cfg = synth.Config("rnd", m, n, kind, min(5, n), 1.0, 2.0, 5.0, alpha, (c,), seed)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    lm = float(np.max(np.abs(oracle.aty(A, b))))
    l1, l2 = c * lm, c * (1 - alpha) * lm / alpha
    with Problem(A, b) as P:
        modes = [("default", {})]
        if P.info("small") == 1:
            modes.append(("graph", {"small": 0}))
        modes += [("host", {"small": 0, "graph": 0}),
                  ("reuse", {"small": 0, "graph": 1, "reuse_min_bytes": 0}),
                  ("reuse-psi-only", {"small": 0, "graph": 1, "reuse_min_bytes": 0, "reuse_frac": 0.0}),
                  ("reuse-host", {"small": 0, "graph": 0, "reuse_min_bytes": 0, "reuse_frac": 0.0})]
        for label, opts in modes:
            for k, v in opts.items():
                P.set_option(k, v)
            compare_to_oracle(A, b, l1, l2, lambda s0, tol, x0: P.solve(l1, l2, s0, tol, x0=x0), sigma0=sigma0,
                              label=f"{label} {case}")
        # a warm-started solve at a smaller λ from that solution (R8: y0 = A x0 − b), graph and host control
        xc, _, _, _ = oracle.solve(A, b, l1, l2, sigma0=sigma0, tol=1e-6)
        w1, w2 = 0.7 * l1, 0.7 * l2
        for graph in (1, 0):
            P.set_option("graph", graph)
            compare_to_oracle(A, b, w1, w2, lambda s0, tol, x0: P.solve(w1, w2, s0, tol, x0=x0), sigma0=sigma0, x0=xc,
                              label=f"warm graph={graph} {case}")
