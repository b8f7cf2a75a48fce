"""Column-sharded solves with device-resident exchanges over peer memory (§8(f3); k_peer.cuh,
ssnal_en_peer_export / _attach).

On one GPU a multi-rank run would need kernels that wait on one another on the same device, which
nothing schedules together, so the multi-rank protocol is tested the way the profiling recipe
prescribes — G ranks emulated as the G CTAs of ONE cooperative launch running the same deposit /
flag / epoch / rank-ordered-sum code (ssnal_en_peer_selftest) — and the solve path at G = 1, where
every exchange kernel runs for real against the rank's own region:
  * graph mode (device-resident control with the exchange kernels inside the conditional bodies) is
    bitwise equal to host-driven control with the same peer kernels and to the host-callback
    provider (set_comm) — iterates, counts and certificates — across the r = 0, SMW-by-gathered-
    columns and m × m-by-summed-Gram branches, warm starts and the factor retry;
  * the results meet the oracle at the BASELINE tolerances (SURVEY §8(c) rule)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import synth
from gpu_util import compare_to_oracle, cuda_ok

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

if cuda_ok():
    from paper_2006_03970_b200 import Problem, SsnalError
    from paper_2006_03970_b200.shard import ThreadGroup, attach_peers
    from paper_2006_03970_b200.ssnal_en import peer_selftest

ARITH = ("status", "outer_iters", "newton_iters", "psi_evals", "backtracks", "aty_passes", "branch_steps", "active",
         "res_kkt1", "res_kkt3", "primal_obj", "dual_obj", "gap", "sigma_final", "jitter_retries")


@pytest.mark.parametrize("G", [1, 2, 3, 8, 16])
@pytest.mark.parametrize("count", [1, 505, 4096])
def test_peer_protocol_emulated_ranks(G, count):
    iters = 31  # 21 small exchanges (consecutive pairs: both parities reused many times) + 10 big
    mis, small, big = peer_selftest(G, iters, count)
    assert mis == 0
    k = np.arange(count, dtype=np.float64)
    q = np.arange(G, dtype=np.float64)[:, None]

    def want(it):  # Σ_q v(q, it, k), v = (q + 1)·1000003 + 7919 it + 31 k (k_peer.cuh)
        return np.sum((q + 1) * 1000003.0 + it * 7919.0 + k[None, :] * 31.0, axis=0)

    last_small = max(it for it in range(iters) if it % 3 != 2)
    last_big = max(it for it in range(iters) if it % 3 == 2)
    for r in range(G):  # every rank holds the same sums
        assert np.array_equal(small[r], want(last_small))
        assert np.array_equal(big[r], want(last_big))


def test_peer_argument_validation():
    cfg = synth.CONFIGS["cfg1"]
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    with Problem(A, b) as P:
        with pytest.raises(SsnalError):
            P.peer_attach(0, 1, [b"\0" * 64])  # no export yet
        with pytest.raises(SsnalError):
            P.peer_export(17)
        h = P.peer_export(2)
        assert len(h) == 64
        with pytest.raises(SsnalError):
            P.peer_attach(0, 1, [h])  # exported for 2 ranks
        with pytest.raises(SsnalError):
            P.peer_attach(2, 2, [h, h])  # rank out of range
    with pytest.raises(SsnalError):
        peer_selftest(0, 1, 1)


def _handles(A, b, kinds):
    """One single-rank sharded handle per kind: 'cb' host-callback provider (host-driven), 'ph' peer
    kernels with host-driven control, 'pg' peer kernels with graph control."""
    out = {}
    for kind in kinds:
        P = Problem(A, b)
        if kind == "cb":
            P.set_comm(ThreadGroup(1).member(0), 0, 1)
        else:
            assert attach_peers(P) == (0, 1)
            P.set_option("graph", 1 if kind == "pg" else 0)
        out[kind] = P
    return out


def _same(a, b, label):
    xa, sa = a
    xb, sb = b
    assert np.array_equal(xa, xb), (label, float(np.max(np.abs(xa - xb))))
    for k in ARITH:
        va, vb = sa[k], sb[k]
        same = (va == vb) or (isinstance(va, float) and np.isnan(va) and np.isnan(vb))
        assert same, (label, k, va, vb)


@pytest.mark.parametrize("name,n", [("cfg2", 20_000), ("cfg3", 20_000), ("cfg1", None), ("cfg4", 12_000)])
def test_peer_graph_equals_host_and_callback(name, n):
    # cfg4 recipe: m = 800 > 512, so the evaluation runs on the 8-CTA-cluster kernels and the exchange
    # record (m + 5 = 805) spans two 32-element blocks per CTA of k_peer_eval
    cfg = synth.CONFIGS[name] if n is None else synth.scaled(synth.CONFIGS[name], n=n)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    lm1 = float(np.max(np.abs(oracle.aty(A, b))))
    lm = lm1 / cfg.alpha
    H = _handles(A, b, ("cb", "ph", "pg"))
    try:
        for P in H.values():
            assert P.lambda_max_l1 == pytest.approx(lm1, rel=1e-13)
        seen = np.zeros(3, dtype=int)
        x = None
        for c in (0.9, 0.3, 0.05):
            l1, l2 = c * cfg.alpha * lm, c * (1 - cfg.alpha) * lm
            res = {k: P.solve(l1, l2, cfg.sigma0, cfg.tol) for k, P in H.items()}
            _same(res["pg"], res["ph"], (name, c, "graph vs host"))
            _same(res["pg"], res["cb"], (name, c, "peer vs callback"))
            seen += np.array(res["pg"][1]["branch_steps"][:3])
            par, stg, stc, _ = compare_to_oracle(A, b, l1, l2,
                                                 lambda s0, tol, x0: H["pg"].solve(l1, l2, s0, tol, x0=x0),
                                                 sigma0=cfg.sigma0, tol=cfg.tol, label=(name, c))
            # warm start from the previous c (y0 = A x0 − b through the exchange)
            if x is not None:
                wr = {k: P.solve(l1, l2, cfg.sigma0, cfg.tol, x0=x) for k, P in H.items()}
                _same(wr["pg"], wr["cb"], (name, c, "warm peer vs callback"))
                _same(wr["pg"], wr["ph"], (name, c, "warm graph vs host"))
            x = res["pg"][0]
        if name in ("cfg2", "cfg3"):
            assert seen[1] > 0 and seen[2] > 0  # the gathered-column SMW and summed-Gram m × m steps ran
    finally:
        for P in H.values():
            P.close()


def test_peer_factor_retry_and_genotypes():
    """The R36 retry inside the graph on a peer handle (injected factor failure), and a packed-genotype
    handle (§8(f4) storage: the gathered columns are decoded by the column accessor)."""
    cfg = synth.scaled(synth.CONFIGS["cfg2"], n=12_000)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    lm = float(np.max(np.abs(oracle.aty(A, b)))) / cfg.alpha
    l1, l2 = 0.2 * cfg.alpha * lm, 0.2 * (1 - cfg.alpha) * lm
    H = _handles(A, b, ("cb", "pg"))
    try:
        for P in H.values():
            P.set_option("test_fail_factor", 1)
        res = {k: P.solve(l1, l2, cfg.sigma0, cfg.tol) for k, P in H.items()}
        assert res["pg"][1]["jitter_retries"] == 1 and res["pg"][1]["status"] == 0
        _same(res["pg"], res["cb"], "retry")
    finally:
        for P in H.values():
            P.close()
    m, n = 300, 9000
    gc = synth.Config("gp", m, n, synth.GENO_STD, 10, 0.1, 0.3, 1.0, 0.5, (0.3,), 19)
    codes, tab = synth.geno_codes(gc)
    Ad = synth.decode_geno(codes, tab, m)
    bg, _ = synth.response(gc)
    lmg = float(np.max(np.abs(oracle.aty(Ad, bg)))) / gc.alpha
    with Problem.from_geno(codes, tab, bg) as P:
        attach_peers(P)
        for c in (0.3, 0.05):
            l1, l2 = c * gc.alpha * lmg, c * (1 - gc.alpha) * lmg
            compare_to_oracle(Ad, bg, l1, l2, lambda s0, tol, x0: P.solve(l1, l2, s0, tol, x0=x0),
                              sigma0=gc.sigma0, tol=gc.tol, label=("geno", c))


def test_peer_path_sigma_carried():
    """A warm-started λ path (σ carried, R38) on a peer handle: point by point equal to the callback
    provider and, per point, parity with the oracle's path."""
    import torch

    cfg = synth.scaled(synth.CONFIGS["cfg2"], n=20_000)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    lm = float(np.max(np.abs(oracle.aty(A, b)))) / cfg.alpha
    cs = list(cfg.cs)
    l1s = [c * cfg.alpha * lm for c in cs]
    l2s = [c * (1 - cfg.alpha) * lm for c in cs]
    H = _handles(A, b, ("cb", "pg"))
    try:
        out = {}
        for k, P in H.items():
            X = torch.zeros((len(cs), cfg.n), dtype=torch.float64, device="cuda")
            sts = P.solve_path_device(l1s, l2s, cfg.sigma0, cfg.tol, 0, X.data_ptr())
            out[k] = (X.cpu().numpy(), sts)
        for i in range(len(cs)):
            _same((out["pg"][0][i], out["pg"][1][i]), (out["cb"][0][i], out["cb"][1][i]), ("path", i))
        orc = oracle.solve_path_lambdas(A, b, list(zip(l1s, l2s)), sigma0=cfg.sigma0, tol=cfg.tol)
        for i, (xc, _, sc) in enumerate(orc):
            xg = out["pg"][0][i]
            Fg = oracle.primal_obj(A, b, xg, l1s[i], l2s[i])
            Fc = oracle.primal_obj(A, b, xc, l1s[i], l2s[i])
            assert abs(Fg - Fc) <= 1e-9 * abs(Fc), (i, Fg, Fc)
            assert abs(out["pg"][1][i]["newton_iters"] - sc["newton_iters"]) <= 1
    finally:
        for P in H.values():
            P.close()


def test_bench_shard_peer_one_gpu():
    """bench.py --shard with the default peer provider: the sharded handle keeps device-resident
    control (graph), and its line says so."""
    env = dict(os.environ, PYTHONPATH=ROOT)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "cfg1", "--shard", "--steps", "2",
                          "--warmup", "3", "--no-cpu", "--no-e2e"], capture_output=True, text=True, env=env, timeout=600,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["scaling"] == "strong" and d["value"] > 0
    assert "peer memory" in d["config"]["parallelism"]
    assert d["config"]["control"].startswith("device-resident")
    assert all(it["outer"] > 0 for it in d["iterations"])
