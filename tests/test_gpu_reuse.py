"""Option reuse_atb (reading R40): a cold solve's first Newton direction is d = −b exactly (x0 = 0 ⇒
y0 = 0, J = ∅, g = b), so the trial product Aᵀ(y0 + d) equals −(Aᵀb) bit for bit — the product
ssnal_en_create forms for λmax and keeps.  K1 then takes w from it instead of streaming A.  The
whole solve must be BITWISE what the streaming launch gives (x and every statistic), in both
control modes, for ragged n / m, with backtracking at the first step, and it must not fire on warm
starts.  Parity with the oracle is held by every other solve test (the option is on by default)."""
import numpy as np
import pytest

import synth
from gpu_util import compare_to_oracle, cuda_ok

pytestmark = pytest.mark.gpu

if cuda_ok():
    from paper_2006_03970_b200 import Problem

SAME = ["status", "outer_iters", "newton_iters", "psi_evals", "backtracks", "aty_passes", "branch_steps",
        "line_search_stalled", "active", "res_kkt1", "res_kkt3", "primal_obj", "dual_obj", "gap", "sigma_final"]


def same_stats(a, b):
    for k in SAME:
        u, v = a[k], b[k]
        assert (u == v) or (isinstance(u, float) and np.isnan(u) and np.isnan(v)), (k, u, v)


def lambdas(alpha, lm, c):
    lmax = lm / alpha
    return c * alpha * lmax, c * (1 - alpha) * lmax


def problem(m, n, seed, k=7):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((n, m))  # (n, m) C-contiguous = column-major m × n (the ABI's layout)
    A -= A.mean(axis=1, keepdims=True)
    A /= A.std(axis=1, keepdims=True)
    xs = np.zeros(n)
    xs[rng.choice(n, size=min(k, n), replace=False)] = rng.uniform(1, 2, min(k, n)) * rng.choice([-1, 1], min(k, n))
    b = xs @ A + 0.3 * rng.standard_normal(m)
    return np.ascontiguousarray(A), b


@pytest.mark.parametrize("m,n", [(50, 1000), (33, 4099), (129, 20011), (500, 30000), (800, 9001), (1024, 2500),
                                 (7, 65)])
@pytest.mark.parametrize("graph", [0, 1])
def test_reuse_is_bitwise_the_streaming_pass(m, n, graph):
    A, b = problem(m, n, 100 + m)
    with Problem(A, b) as P:
        P.set_option("small", 0)
        P.set_option("graph", graph)
        assert P.info("reuse_atb") == 1
        P.set_option("reuse_frac", 1.0)  # no gate: reuse whatever the first active set (the worst case for the gather)
        P.set_option("reuse_min_bytes", 0)  # the default skips the gate (and its sync) for designs below 2 GB
        lm = P.lambda_max_l1
        for c in (0.6, 0.15):
            l1, l2 = lambdas(0.7, lm, c)
            P.set_option("reuse_atb", 1)
            n0 = P.info("atb_reuses")
            x1, s1 = P.solve(l1, l2, 5e-3, 1e-6)
            assert P.info("atb_reuses") == n0 + 1
            P.set_option("reuse_atb", 0)
            x0, s0 = P.solve(l1, l2, 5e-3, 1e-6)
            assert P.info("atb_reuses") == n0 + 1
            assert s1["status"] == 0 and s1["newton_iters"] >= 1
            assert np.array_equal(x1, x0), np.max(np.abs(x1 - x0))
            same_stats(s1, s0)


def test_reuse_with_backtracking_at_the_first_step():
    """μ close to ½ forces halvings of the first step: the backtracks read w + s(w1 − w) with w1 the
    reused product, so w1 must be materialised exactly as the streaming pass writes it."""
    A, b = problem(200, 15000, 5)
    for graph in (0, 1):
        with Problem(A, b) as P:
            P.set_option("small", 0)
            P.set_option("graph", graph)
            P.set_option("mu", 0.49)
            P.set_option("reuse_frac", 1.0)
            P.set_option("reuse_min_bytes", 0)
            l1, l2 = lambdas(0.5, P.lambda_max_l1, 0.1)
            x1, s1 = P.solve(l1, l2, 5e-3, 1e-6)
            P.set_option("reuse_atb", 0)
            x0, s0 = P.solve(l1, l2, 5e-3, 1e-6)
            assert s1["backtracks"] > 0
            assert np.array_equal(x1, x0)
            same_stats(s1, s0)


def test_reuse_not_used_on_warm_starts_and_matches_oracle():
    cfg = synth.scaled(synth.CONFIGS["cfg3"], n=20000)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    with Problem(A, b) as P:
        P.set_option("reuse_min_bytes", 0)
        lm = P.lambda_max_l1
        l1, l2 = lambdas(cfg.alpha, lm, 0.6)
        compare_to_oracle(A, b, l1, l2, lambda s0, tol, x0: P.solve(l1, l2, s0, tol, x0=x0), cfg.sigma0, cfg.tol)
        xg, sg = P.solve(l1, l2, cfg.sigma0, cfg.tol)
        n0 = P.info("atb_reuses")
        assert n0 >= 1
        l1b, l2b = lambdas(cfg.alpha, lm, 0.5)
        xw, sw = P.solve(l1b, l2b, cfg.sigma0, cfg.tol, x0=xg)  # warm: y0 = A x0 − b, no reuse
        assert P.info("atb_reuses") == n0 and sw["status"] == 0
        # x = 0 at λ1 = ‖Aᵀb‖∞: the single Newton step's trial is the reused product
        x0, s0 = P.solve(lm, 0.0, cfg.sigma0, cfg.tol)
        assert np.all(x0 == 0) and s0["newton_iters"] == 1


def test_gate_follows_the_first_active_set():
    """The reused launch gathers the first trial's active columns {|Aᵀb|_i > λ1} from global memory, so
    the default gate (reuse_frac = 0.3) uses it only while that set is small; either way the result is
    the same bits."""
    A, b = problem(100, 40000, 11)
    atb = np.abs(A @ b)
    with Problem(A, b) as P:
        P.set_option("small", 0)
        P.set_option("reuse_min_bytes", 0)
        P.set_option("reuse_psi_only", 0)  # above the gate: stream (the ψ-only mode has its own test below)
        lm = P.lambda_max_l1
        for c, alpha in ((0.9, 0.7), (0.05, 0.7)):
            l1, l2 = lambdas(alpha, lm, c)
            expect = int(np.count_nonzero(atb > l1) <= int(0.3 * P.n))
            res = []
            for graph in (0, 1):
                P.set_option("graph", graph)
                n0 = P.info("atb_reuses")
                res.append(P.solve(l1, l2, 5e-3, 1e-6))
                assert P.info("atb_reuses") == n0 + expect, (c, graph)
            assert np.array_equal(res[0][0], res[1][0])
            same_stats(res[0][1], res[1][1])
        assert np.count_nonzero(atb > lambdas(0.7, lm, 0.05)[0]) > int(0.3 * P.n)  # the second case was gated off


def test_small_designs_skip_the_gate():
    """Below reuse_min_bytes (2 GB of A) a pass costs less than the gate's synchronisation: no gate."""
    A, b = problem(100, 5000, 3)
    with Problem(A, b) as P:
        P.set_option("small", 0)
        l1, l2 = lambdas(0.7, P.lambda_max_l1, 0.9)
        x, st = P.solve(l1, l2, 5e-3, 1e-6)
        assert st["status"] == 0 and P.info("atb_reuses") == 0


def test_reuse_on_sharded_handles():
    """Column-sharded handles (§8(f3)): every rank gates on its own block (the decision only changes
    which K1 instantiation runs, never a bit of the result), through the host-callback provider with
    2 shards, and through the peer-kernel provider in both control modes."""
    from paper_2006_03970_b200.shard import ThreadGroup, attach_peers, column_range, run_threads

    cfg = synth.scaled(synth.CONFIGS["cfg3"], n=12000)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    with Problem(A, b) as P:
        P.set_option("small", 0)
        lm = P.lambda_max_l1
        l1, l2 = lambdas(cfg.alpha, lm, 0.6)
        P.set_option("reuse_atb", 0)
        xref, sref = P.solve(l1, l2, cfg.sigma0, cfg.tol)
    # peer provider (G = 1, real exchange kernels), host-driven and graph control
    for graph in (0, 1):
        with Problem(A, b) as P:
            assert attach_peers(P) == (0, 1)
            P.set_option("graph", graph)
            P.set_option("reuse_min_bytes", 0)
            x1, s1 = P.solve(l1, l2, cfg.sigma0, cfg.tol)
            assert P.info("atb_reuses") == 1
            P.set_option("reuse_atb", 0)
            x0, s0 = P.solve(l1, l2, cfg.sigma0, cfg.tol)
            assert np.array_equal(x1, x0)
            same_stats(s1, s0)
            assert np.max(np.abs(x1 - xref)) <= 1e-9 * np.max(np.abs(xref))
    # two shards, one thread each, host callbacks
    G = 2
    grp = ThreadGroup(G)
    shards = []
    for q in range(G):
        j0, j1 = column_range(A.shape[0], q, G)
        shards.append(Problem(np.ascontiguousarray(A[j0:j1]), b))
    run_threads([(lambda q=q: shards[q].set_comm(grp.member(q), q, G)) for q in range(G)], grp)
    outs = {}
    for on in (1, 0):
        for S in shards:
            S.set_option("reuse_atb", on)
            S.set_option("reuse_min_bytes", 0)
        res = run_threads([(lambda q=q: shards[q].solve(l1, l2, cfg.sigma0, cfg.tol)) for q in range(G)], grp)
        outs[on] = (np.concatenate([r[0] for r in res]), res[0][1])
    assert sum(S.info("atb_reuses") for S in shards) >= 1
    assert np.array_equal(outs[1][0], outs[0][0])
    same_stats(outs[1][1], outs[0][1])
    for S in shards:
        S.close()


@pytest.mark.parametrize("m,n", [(800, 6000), (203, 9001), (64, 2048)])
@pytest.mark.parametrize("graph", [0, 1])
def test_reuse_on_packed_genotypes(m, n, graph):
    """K1g's REUSE instantiation (packed 2-bit codes, §8(f4)): Aᵀ(−b) = −(Aᵀb) bitwise there too (the
    fixed-point rounding of y is odd), the ∇ψ rows decoded from the active columns' codes."""
    cfg = synth.scaled(synth.CONFIGS["cfg4"], n=n, m=m)
    codes, tab = synth.geno_codes(cfg)
    b, _ = synth.response(cfg)
    with Problem.from_geno(codes, tab, b) as P:
        P.set_option("small", 0)
        P.set_option("graph", graph)
        P.set_option("reuse_frac", 1.0)
        P.set_option("reuse_min_bytes", 0)
        assert P.info("reuse_atb") == 1
        lm = P.lambda_max_l1
        for c in (0.6, 0.2):
            l1, l2 = lambdas(cfg.alpha, lm, c)
            P.set_option("reuse_atb", 1)
            n0 = P.info("atb_reuses")
            x1, s1 = P.solve(l1, l2, cfg.sigma0, cfg.tol)
            assert P.info("atb_reuses") == n0 + 1
            P.set_option("reuse_atb", 0)
            x0, s0 = P.solve(l1, l2, cfg.sigma0, cfg.tol)
            assert s1["status"] == 0 and s1["newton_iters"] >= 1
            assert np.array_equal(x1, x0), np.max(np.abs(x1 - x0))
            same_stats(s1, s0)


def test_psi_only_trials_and_the_streamed_redo():
    """Above reuse_frac the trial at y = −b is served ψ-only (no ∇ψ rows: most columns are active there);
    Armijo usually rejects s = 1 and the gradient is rebuilt at the accepted step, else the trial is redone
    streamed.  Both outcomes must give the bits of the plain solve, in both control modes: small λ (large
    active set, s = 1 rejected) and λ near λmax with reuse_frac = 0 (ψ-only although J is tiny: s = 1 is
    accepted, the redo runs)."""
    A, b = problem(120, 30000, 21)
    for graph in (0, 1):
        with Problem(A, b) as P:
            P.set_option("small", 0)
            P.set_option("graph", graph)
            P.set_option("reuse_min_bytes", 0)
            lm = P.lambda_max_l1
            seen = {"rejected": 0, "accepted": 0}
            for c, frac in ((0.05, 0.3), (0.02, 0.3), (0.9, 0.0), (0.6, 0.0), (0.3, 0.0)):
                l1, l2 = lambdas(0.7, lm, c)
                P.set_option("reuse_frac", frac)
                P.set_option("reuse_atb", 1)
                n0 = P.info("atb_reuses")
                x1, s1 = P.solve(l1, l2, 5e-3, 1e-6)
                assert P.info("atb_reuses") == n0 + 1
                P.set_option("reuse_atb", 0)
                x0, s0 = P.solve(l1, l2, 5e-3, 1e-6)
                assert np.array_equal(x1, x0), (c, graph, np.max(np.abs(x1 - x0)))
                same_stats(s1, s0)
                seen["rejected" if s1["backtracks"] > 0 else "accepted"] += 1
            assert seen["rejected"] > 0 and seen["accepted"] > 0, seen
            # reuse_psi_only = 0: above the gate the solve streams
            P.set_option("reuse_atb", 1)
            P.set_option("reuse_psi_only", 0)
            n0 = P.info("atb_reuses")
            P.solve(l1, l2, 5e-3, 1e-6)
            assert P.info("atb_reuses") == n0


def test_reuse_with_a_deeper_k1_ring():
    """Option k1_stages changes the dynamic shared memory of both K1 instantiations (a larger ring than
    the one configured at create must not make the REUSE launch fail)."""
    A, b = problem(64, 9000, 31)  # small stages: the default ring is far below 224 KB, 16 stages still fit
    with Problem(A, b) as P:
        P.set_option("small", 0)
        P.set_option("reuse_min_bytes", 0)
        l1, l2 = lambdas(0.7, P.lambda_max_l1, 0.5)
        x0, s0 = P.solve(l1, l2, 5e-3, 1e-6)
        P.set_option("k1_stages", 16)
        for graph in (1, 0):
            P.set_option("graph", graph)
            x1, s1 = P.solve(l1, l2, 5e-3, 1e-6)
            assert np.array_equal(x1, x0)
            same_stats(s1, s0)
