"""Column-sharded solves: rank q of G owns a contiguous block of columns of A,
and the library sums every cross-column quantity over the ranks (the exchange points are listed at
ssnal_en_set_comm in include/ssnal_en.h).

Exchange providers:
  * `attach_peers(problem, group)` — the default for one process per GPU: device-resident exchanges
    over peer memory inside the library (ssnal_en_peer_export / _attach: CUDA IPC regions, P2P
    stores over NVLink, rank-ordered sums), so sharded solves keep the graph's device-resident
    control; torch.distributed only carries the 64-byte IPC handles once;
  * `torch_allreduce(group)` — a host callback per exchange over torch.distributed (NCCL on GPUs;
    gloo on CPU for the host-side tests), stream-ordered with the library's stream (host-driven
    control);
  * `ThreadGroup(G)` — G shards of one problem on one device in one process, one thread each,
    summing through host barriers (a test harness: the kernels of different shards never wait on
    one another; the threads synchronise on the host).

This module is argument marshalling and host synchronisation only; every arithmetic step of the
path runs in the library's kernels (the reductions here are the all-reduce itself)."""
import threading

import torch

SUM, MAX = 0, 1


def column_range(n: int, rank: int, nranks: int):
    """Columns [j0, j1) owned by `rank`: contiguous, sizes differ by at most one."""
    return n * rank // nranks, n * (rank + 1) // nranks


class _Cai:
    """A raw device (or host) pointer viewed as a float64 vector through the CUDA array interface
    (or the numpy array interface on the CPU), so torch can wrap it without a copy."""

    def __init__(self, ptr: int, count: int, device: str):
        iface = {"shape": (int(count),), "typestr": "<f8", "data": (int(ptr), False), "version": 2}
        if device == "cuda":
            self.__cuda_array_interface__ = iface
        else:
            self.__array_interface__ = dict(iface, version=3)


def as_tensor(ptr: int, count: int, device: str = "cuda") -> torch.Tensor:
    if device == "cuda":
        return torch.as_tensor(_Cai(ptr, count, device), device="cuda")
    import numpy as np

    return torch.from_numpy(np.asarray(_Cai(ptr, count, device)))


def exchange_handles(handle: bytes, group=None):
    """All-gather every rank's exchange-region handle in rank order (torch.distributed when it is
    initialised, else a single rank)."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return 0, 1, [handle]
    rank, size = dist.get_rank(group), dist.get_world_size(group)
    out = [None] * size
    dist.all_gather_object(out, handle, group=group)
    return rank, size, out


def attach_peers(problem, group=None):
    """Make `problem` (this rank's column block) a rank of a sharded solve with device-resident
    exchanges over peer memory: export its exchange region, all-gather the IPC handles, attach."""
    import torch.distributed as dist

    size = dist.get_world_size(group) if (dist.is_available() and dist.is_initialized()) else 1
    rank, size, handles = exchange_handles(problem.peer_export(size), group)
    problem.peer_attach(rank, size, handles)
    return rank, size


def torch_allreduce(group=None, device: str = "cuda"):
    """An all-reduce for Problem.set_comm over a torch.distributed group.  NCCL: in place on the device,
    ordered on the library's stream.  Other backends (gloo) with device buffers: staged through host
    memory — the library's stream is drained, the buffer is copied to the host on that stream, reduced
    by the backend on CPU tensors, and copied back on the same stream, so the exchange is complete and
    ordered before the library's next kernel."""
    import torch.distributed as dist

    ops = {SUM: dist.ReduceOp.SUM, MAX: dist.ReduceOp.MAX}
    nccl = device == "cuda" and dist.get_backend(group) == "nccl"

    def fn(buf, count, op, stream):
        t = as_tensor(buf, count, device)
        if device != "cuda":
            dist.all_reduce(t, op=ops[op], group=group)
            return
        # the library's stream; a NULL handle is the legacy default stream, which torch names
        # default_stream() (wrapping it as ExternalStream(0) raced in the two-process test)
        st = torch.cuda.ExternalStream(stream) if stream else torch.cuda.default_stream()
        if nccl:
            with torch.cuda.stream(st):
                dist.all_reduce(t, op=ops[op], group=group)
        else:
            st.synchronize()  # the producing kernels are done
            h = t.to("cpu")
            dist.all_reduce(h, op=ops[op], group=group)
            t.copy_(h)
            torch.cuda.current_stream().synchronize()  # complete before the library's next kernel

    return fn


class ThreadGroup:
    """In-process all-reduce over G shards driven by G threads on one device (tests).  Every
    shard computes the same sum in the same order (shard 0 + 1 + … + G−1), so all shards hold
    bitwise-identical results, as with a real all-reduce."""

    def __init__(self, size: int):
        self.size = size
        self.barrier = threading.Barrier(size)
        self.slots = [None] * size

    def member(self, rank: int):
        def fn(buf, count, op, stream):
            st = torch.cuda.ExternalStream(stream) if stream else torch.cuda.default_stream()
            st.synchronize()
            t = as_tensor(buf, count)
            self.slots[rank] = t.clone()
            torch.cuda.current_stream().synchronize()
            self.barrier.wait()
            acc = self.slots[0].clone()
            for q in range(1, self.size):
                acc = acc + self.slots[q] if op == SUM else torch.maximum(acc, self.slots[q])
            t.copy_(acc)
            torch.cuda.current_stream().synchronize()
            self.barrier.wait()

        return fn


def run_threads(fns, group: "ThreadGroup | None" = None):
    """Run one callable per shard in its own thread; return their results (re-raise the first
    error, after releasing the other shards from the group's barrier)."""
    out = [None] * len(fns)
    err = []

    def wrap(i, f):
        try:
            out[i] = f()
        except BaseException as e:  # noqa: BLE001 - surfaced to the caller below
            err.append(e)
            if group is not None:
                group.barrier.abort()

    ths = [threading.Thread(target=wrap, args=(i, f)) for i, f in enumerate(fns)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    if err:
        raise err[0]
    return out
