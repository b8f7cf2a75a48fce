"""CPU checks of bench.py's host logic: the reference arm (the oracle, this tier's reference),
its single-line output under torchrun with 2 ranks, and the max-over-ranks reduction on gloo."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _json_lines(out):
    return [json.loads(l) for l in out.splitlines() if l.strip().startswith("{")]


def test_reference_arm_single():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "cfg1", "--steps", "1",
                          "--warmup", "1"], cwd=ROOT, capture_output=True, text=True, check=True, timeout=300).stdout
    lines = _json_lines(out)
    assert len(lines) == 1
    d = lines[0]
    assert d["impl"] == "reference" and d["higher_is_better"] is False and d["unit"] == "s"
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_reference_arm_torchrun_two_ranks():
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), "bench.py", "--impl", "reference", "--gpus", "2", "--config",
           "cfg1", "--steps", "1", "--warmup", "1"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1 and lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2


def _worker(rank, world, port, q):
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    import bench

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    q.put((rank, bench.max_over_ranks(1.5 + rank, device="cpu")))
    dist.destroy_process_group()


def test_max_over_ranks_gloo():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res == {0: 2.5, 1: 2.5}


def test_max_over_ranks_without_group():
    sys.path.insert(0, ROOT)
    import bench

    assert bench.max_over_ranks(3.25, device="cpu") == 3.25


def test_small_roofline_line():
    """The single-launch small-problem path has no K1 launches: the bench reports a latency-bound roofline
    for k_small_cl with the effective A-pass bandwidth (passes × 8mn bytes / device time) against the HBM peak."""
    sys.path.insert(0, ROOT)
    import bench

    sts = [{"aty_passes": 16}, {"aty_passes": 4}]
    r = bench.small_roofline(50, 1000, sts, 1e-3, 6500.0, "measured")
    assert r["bound"] == "latency" and r["kernel"] == "k_small_cl" and r["unit"] == "GB/s"
    assert r["bytes_per_launch"] == 20 * 8 * 50 * 1000
    assert r["achieved"] == pytest.approx(20 * 8 * 50 * 1000 / 1e-3 / 1e9)
    assert r["frac"] == pytest.approx(r["achieved"] / 6500.0) and r["launches"] == 2


def test_cpu_leg_parity_block(tmp_path):
    """The clean-process oracle leg of bench.py (cpu_baseline + the §8(d) parity block): fed the oracle's
    own solutions as the 'GPU' solutions, every parity metric is exact; fed a perturbed x, it flags it."""
    sys.path.insert(0, ROOT)
    import numpy as np

    import bench
    import oracle
    import synth

    cfg = synth.CONFIGS["cfg1"]
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    lm = oracle.lambda_max_l1(A, b)
    xs, sts = [], []
    for c in cfg.cs:
        l1, l2 = bench.lambdas(cfg, lm, c)
        x, _, st, _ = oracle.solve(A, b, l1, l2, sigma0=cfg.sigma0, tol=cfg.tol)
        xs.append(x)
        sts.append(st)
    for bad in (False, True):
        d = tmp_path / ("bad" if bad else "ok")
        d.mkdir()
        xg = np.array(xs)
        if bad:
            xg[0, np.argmax(np.abs(xg[0]))] *= 1.01
        np.save(d / "x_gpu.npy", xg)
        np.save(d / "w_gpu.npy", oracle.aty(A, synth.normals(cfg.seed, 12, cfg.m)))
        json.dump([{k: s[k] for k in ("outer_iters", "newton_iters", "active", "status")} for s in sts],
                  open(d / "gpu_stats.json", "w"))
        bench.cpu_leg(str(d), "cfg1")
        out = json.load(open(d / "cpu.json"))
        cb, par = out["cpu_baseline"], out["parity"]
        assert cb["kind"] == "oracle" and cb["value"] > 0 and cb["threads"] >= 1
        assert par["aty_max_scaled_err"] == 0.0
        p0 = par["points"][0]
        assert p0["outer"][0] == p0["outer"][1] and p0["newton"][0] == p0["newton"][1]
        if bad:
            assert not par["ok"] and p0["xinf_rel"] > 1e-3
        else:
            assert par["ok"] and p0["obj_rel"] == 0.0 and p0["xinf_rel"] == 0.0 and p0["J_equal"]


def test_read_ceiling_context():
    """The roofline line's read-ceiling context is the best GB/s of the committed read probe."""
    import json
    import sys

    sys.path.insert(0, ROOT)
    import bench

    p = os.path.join(ROOT, "profiles", "r2_read_ceiling_probe.jsonl")
    best = 0.0
    for line in open(p):
        try:
            best = max(best, float(json.loads(line).get("GBps", 0.0)))
        except ValueError:
            pass
    assert bench._read_ceiling() == best and best > 7000.0
