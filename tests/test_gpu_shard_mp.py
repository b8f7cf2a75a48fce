"""Column-sharded solve with ONE PROCESS PER RANK, as a multi-GPU run is launched:
2 processes (torch.multiprocessing spawn, rendezvous on 127.0.0.1), each owning a contiguous column
block of A in its own handle, exchanging through torch.distributed (gloo backend, CUDA tensors — the
same `torch_allreduce` provider the NCCL ranks of `bench.py --shard` use).  This box has one GPU, so
both processes share it; their kernels never wait on one another (every exchange is a host-side
collective between the ranks' streams), so nothing here depends on co-residency.  The assembled
warm-started path (σ carried, R38) is compared with the oracle on the full design: solution parity
at the BASELINE tolerances, iteration counts (±1 rule), identical statistics on both ranks."""
import os
import socket
import sys

import numpy as np
import pytest

import oracle
import synth
from gpu_util import cuda_ok, solution_parity

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CS = {"cfg2": (0.9, 0.4, 0.1), "cfg3": (0.5, 0.2, 0.05)}  # SMW (gathered columns) and m × m (summed Grams) steps


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, cfg_args, q):
    try:
        sys.path.insert(0, ROOT)
        import torch
        import torch.distributed as dist

        import synth as sy
        from paper_2006_03970_b200 import Problem
        from paper_2006_03970_b200.shard import column_range, torch_allreduce

        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        cfg = sy.scaled(sy.CONFIGS[cfg_args[0]], n=cfg_args[1])
        j0, j1 = column_range(cfg.n, rank, world)
        A = sy.design(cfg, j0, j1)
        b, _ = sy.response(cfg)
        out = []
        with Problem(A, b) as P:
            P.set_comm(torch_allreduce(device="cuda"), rank, world)
            lm = P.lambda_max_l1 / cfg.alpha  # the global ‖Aᵀb‖∞ (max over ranks)
            x, sig = None, cfg.sigma0
            for c in CS[cfg_args[0]]:
                l1, l2 = c * cfg.alpha * lm, c * (1 - cfg.alpha) * lm
                x, st = P.solve(l1, l2, sig, cfg.tol, x0=x)
                sig = st["sigma_final"]
                out.append((x.copy(), st))
        q.put((rank, j0, j1, out, None))
        dist.destroy_process_group()
    except BaseException as e:  # noqa: BLE001 - reported to the parent
        import traceback

        q.put((rank, 0, 0, None, traceback.format_exc()))


@pytest.mark.parametrize("name,n", [("cfg2", 20_000), ("cfg3", 30_000)])
def test_two_process_sharded_path(name, n):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, (name, n), q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r, j0, j1, out, err = q.get(timeout=600)
        assert err is None, err
        res[r] = (j0, j1, out)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    cfg = synth.scaled(synth.CONFIGS[name], n=n)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    lm = oracle.lambda_max_l1(A, b) / cfg.alpha
    ls = [(c * cfg.alpha * lm, c * (1 - cfg.alpha) * lm) for c in CS[name]]
    orc = oracle.solve_path_lambdas(A, b, ls, sigma0=cfg.sigma0, tol=cfg.tol)
    seen = np.zeros(3, dtype=int)
    for i, ((l1, l2), (xc, _, sc)) in enumerate(zip(ls, orc)):
        s0, s1 = res[0][2][i][1], res[1][2][i][1]
        for key in ("status", "outer_iters", "newton_iters", "active", "res_kkt1", "res_kkt3", "primal_obj",
                    "dual_obj", "sigma_final", "branch_steps"):
            assert s0[key] == s1[key], key  # identical reduced values → identical decisions on both ranks
        x = np.concatenate([res[0][2][i][0], res[1][2][i][0]])
        assert s0["status"] == 0 and sc["status"] == 0
        assert abs(s0["outer_iters"] - sc["outer_iters"]) <= 1 and abs(s0["newton_iters"] - sc["newton_iters"]) <= 1
        par = solution_parity(x, xc, oracle.primal_obj(A, b, x, l1, l2), oracle.primal_obj(A, b, xc, l1, l2))
        assert par["ok"], (i, par, s0, sc)
        assert s0["primal_obj"] == pytest.approx(oracle.primal_obj(A, b, x, l1, l2), rel=1e-12)
        seen += np.array(s0["branch_steps"][:3])
    assert seen[1] > 0 and (name != "cfg3" or seen[2] > 0)
