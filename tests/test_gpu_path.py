"""The λ-path call ssnal_en_solve_path_device (BASELINE configs[1]'s warm-started path):
every point enqueued before one synchronisation must give exactly the loop of single device solves
(same kernels in the same order: x bitwise, statistics equal), in graph mode, on the one-CTA path, and
through the host-driven fallback; a cold first point and an x0 start; bad arguments are EINVAL."""
import numpy as np
import pytest

import synth
from gpu_util import cuda_ok

pytestmark = pytest.mark.gpu

if cuda_ok():
    import torch
    from paper_2006_03970_b200 import Problem, SsnalError

KEYS = ["status", "outer_iters", "newton_iters", "psi_evals", "backtracks", "aty_passes", "branch_steps",
        "line_search_stalled", "active", "res_kkt1", "res_kkt3", "primal_obj", "dual_obj", "gap", "sigma_final",
        "jitter_retries", "cg_iters", "kernel_launches"]


def loop_vs_path(P, ls, sigma0, tol, n, x0=None):
    k = len(ls)
    xl = torch.empty((k, n), dtype=torch.float64, device="cuda")
    sl = []
    for i, (l1, l2) in enumerate(ls):
        x0p = (x0.data_ptr() if x0 is not None else 0) if i == 0 else xl[i - 1].data_ptr()
        sl.append(P.solve_device(l1, l2, sigma0, tol, x0p, xl[i].data_ptr()))
    xp = torch.empty((k, n), dtype=torch.float64, device="cuda")
    sp = P.solve_path_device([a for a, _ in ls], [b for _, b in ls], sigma0, tol,
                             x0.data_ptr() if x0 is not None else 0, xp.data_ptr())
    torch.cuda.synchronize()
    assert torch.equal(xl, xp)
    for a, b in zip(sl, sp):
        for key in KEYS:
            assert a[key] == b[key] or (isinstance(a[key], float) and np.isnan(a[key]) and np.isnan(b[key])), key
        assert b["time_device_s"] > 0


@pytest.mark.parametrize("name,n,graph", [("cfg2", 20_000, 1), ("cfg2", 20_000, 0), ("cfg1", None, 1)])
def test_path_matches_loop(name, n, graph):
    cfg = synth.CONFIGS[name] if n is None else synth.scaled(synth.CONFIGS[name], n=n)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    with Problem(A, b) as P:
        P.set_option("graph", graph)
        lm = P.lambda_max_l1 / cfg.alpha
        cs = np.linspace(0.9, 0.1, 10)
        ls = [(c * cfg.alpha * lm, c * (1 - cfg.alpha) * lm) for c in cs]
        loop_vs_path(P, ls, cfg.sigma0, cfg.tol, A.shape[0])
        # a warm first point from a given x0
        x0 = torch.zeros(A.shape[0], dtype=torch.float64, device="cuda")
        x0[3] = 0.1
        loop_vs_path(P, ls[:3], cfg.sigma0, cfg.tol, A.shape[0], x0=x0)
        with pytest.raises(SsnalError):
            P.solve_path_device([ls[0][0], -1.0], [ls[0][1], 1.0], cfg.sigma0, cfg.tol, 0,
                                torch.empty((2, A.shape[0]), dtype=torch.float64, device="cuda").data_ptr())
