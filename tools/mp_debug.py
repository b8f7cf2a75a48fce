"""Debug the two-process sharded solve: log every exchange (count, op, checksum before/after) per rank."""
import os
import socket
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _rank(rank, world, port):
    import numpy as np
    import torch
    import torch.distributed as dist

    import synth as sy
    from paper_2006_03970_b200 import Problem
    from paper_2006_03970_b200.shard import as_tensor, column_range, torch_allreduce

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    cfg = sy.scaled(sy.CONFIGS["cfg2"], n=20000)
    j0, j1 = column_range(cfg.n, rank, world)
    A = sy.design(cfg, j0, j1)
    b, _ = sy.response(cfg)
    base = torch_allreduce(device="cuda")
    log = open(f"gpurun_out/mpdbg_{rank}.log", "w")
    k = [0]

    sync = os.environ.get("MPDBG_SYNC", "0") == "1"

    def fn(buf, count, op, stream):
        if sync:
            torch.cuda.synchronize()
        base(buf, count, op, stream)
        u = as_tensor(buf, count).cpu().numpy().copy()
        log.write(f"{k[0]} count={count} op={op} after_sum={u.sum():.17g} head={u[:3].tolist()}\n")
        log.flush()
        k[0] += 1

    with Problem(A, b) as P:
        P.set_comm(fn, rank, world)
        lm = P.lambda_max_l1 / cfg.alpha
        x, sig = None, cfg.sigma0
        for c in (0.9, 0.4, 0.1):
            l1, l2 = c * cfg.alpha * lm, c * (1 - cfg.alpha) * lm
            x, st = P.solve(l1, l2, sig, cfg.tol, x0=x)
            sig = st["sigma_final"]
            log.write(f"SOLVE c={c} {st}\n")
    dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    ps = [ctx.Process(target=_rank, args=(r, 2, port)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=300)
    print([p.exitcode for p in ps])
