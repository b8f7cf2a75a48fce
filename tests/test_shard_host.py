"""Host side of the column-sharded path without a GPU: the column partition,
and the torch.distributed all-reduce provider that ssnal_en_set_comm calls, run on gloo with
world size 2 over raw host pointers (the same callable the GPU ranks use with NCCL), including
the sum/max ops and the exchange-record layout [vector | 4 scalars | r]."""
import os
import socket
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_column_range_partitions():
    sys.path.insert(0, ROOT)
    from paper_2006_03970_b200.shard import column_range

    for n, G in [(10, 3), (100_000, 8), (7, 7), (5, 1), (1_000_003, 4)]:
        rs = [column_range(n, q, G) for q in range(G)]
        assert rs[0][0] == 0 and rs[-1][1] == n
        assert all(rs[q][1] == rs[q + 1][0] for q in range(G - 1))
        sizes = [b - a for a, b in rs]
        assert max(sizes) - min(sizes) <= 1


def _worker(rank, world, port, q):
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    from paper_2006_03970_b200.shard import MAX, SUM, torch_allreduce

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    fn = torch_allreduce(device="cpu")
    m = 37
    # an exchange record: partial A_J P_J (m), 4 scalar partials, the local active count
    rec = np.concatenate([np.arange(m, dtype=np.float64) * (rank + 1), [1.0 + rank, 2.0, 3.0, 4.0 * rank], [10.0 + rank]])
    fn(rec.ctypes.data, rec.size, SUM, 0)
    lm = np.array([3.0 + 5.0 * rank])
    fn(lm.ctypes.data, 1, MAX, 0)
    q.put((rank, rec.tolist(), float(lm[0])))
    dist.destroy_process_group()


def test_torch_allreduce_gloo_world2():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r, rec, lm = q.get(timeout=120)
        res[r] = (rec, lm)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    m = 37
    want = np.concatenate([np.arange(m) * 3.0, [3.0, 4.0, 6.0, 4.0], [21.0]])
    for r in (0, 1):
        assert np.array_equal(np.array(res[r][0]), want)  # sums, identical on both ranks
        assert res[r][1] == 8.0  # max


class _FakeProblem:
    """Stands in for a Problem in the handle exchange of shard.attach_peers (no GPU): records the
    export size and the handles it is attached with."""

    def __init__(self, rank):
        self.rank = rank
        self.exported = None
        self.attached = None

    def peer_export(self, nranks):
        self.exported = nranks
        return bytes([self.rank + 1]) * 64  # a distinct 64-byte "IPC handle" per rank

    def peer_attach(self, rank, nranks, handles):
        self.attached = (rank, nranks, [bytes(h) for h in handles])


def _attach_worker(rank, world, port, q):
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    from paper_2006_03970_b200.shard import attach_peers

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    P = _FakeProblem(rank)
    ret = attach_peers(P)
    q.put((rank, ret, P.exported, P.attached))
    dist.destroy_process_group()


def test_attach_peers_exchanges_handles_gloo_world2():
    """shard.attach_peers (the device-resident exchange provider, ssnal_en_peer_export / _attach):
    every rank exports a region sized for the world, receives every rank's IPC handle in rank order
    and attaches as its own rank."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_attach_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r, ret, exported, attached = q.get(timeout=120)
        res[r] = (ret, exported, attached)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in (0, 1):
        ret, exported, attached = res[r]
        assert ret == (r, 2) and exported == 2
        assert attached == (r, 2, [bytes([1]) * 64, bytes([2]) * 64])


def test_attach_peers_single_process():
    """Without torch.distributed the handle is a one-rank group."""
    sys.path.insert(0, ROOT)
    from paper_2006_03970_b200.shard import attach_peers

    P = _FakeProblem(0)
    assert attach_peers(P) == (0, 1)
    assert P.exported == 1 and P.attached == (0, 1, [bytes([1]) * 64])
