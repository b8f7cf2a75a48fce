"""bench.py's multi-rank code paths (the driver's `torchrun --nproc-per-node N bench.py --gpus N` launch),
exercised on a one-GPU box: with the test hook BENCH_TEST_ONE_DEVICE=1 every rank uses device 0 and the
group is gloo (NCCL refuses two ranks on one device).  Replicas (each rank its own cfg2 path) and
--shard (the ranks split the columns of one problem, exchanging through the all-reduce provider):
exactly one JSON line from rank 0 with n_gpus = 2, and the same iterations as a single rank."""
import json
import os
import socket
import subprocess
import sys

import pytest

from gpu_util import cuda_ok

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(extra):
    env = dict(os.environ, BENCH_TEST_ONE_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2", "--config", "cfg2", "--steps", "2",
           "--warmup", "3", "--no-cpu", "--no-e2e"] + extra
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return lines[0]


@pytest.mark.parametrize("mode", ["replicas", "shard"])
def test_bench_two_ranks(mode):
    d = _run(["--shard"] if mode == "shard" else [])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["scaling"] == ("strong" if mode == "shard" else "weak")
    its = [(i["outer"], i["newton"], i["r"]) for i in d["iterations"]]
    assert len(its) == 10 and all(o >= 1 for o, _, _ in its)
    assert its[-1][2] == 391  # the c = 0.1 support of the single-rank path (profiles/r2_bench_cfg2.json)
