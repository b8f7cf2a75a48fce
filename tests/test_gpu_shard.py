"""Column-sharded solves on one GPU: G shards of one problem, one handle and
one thread each, exchanging through an in-process all-reduce (shard.ThreadGroup).  The assembled
solution against the single-handle solve and the oracle, across c values that exercise the r = 0,
SMW-by-gathered-columns and m × m-by-summed-Gram branches, warm starts (including shards without
an x0 slice), λmax, the objective and statistics, and the factor retry."""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import cuda_ok, solution_parity

pytestmark = pytest.mark.gpu

if cuda_ok():
    from paper_2006_03970_b200 import Problem, SsnalError
    from paper_2006_03970_b200.shard import ThreadGroup, column_range, run_threads


def make_shards(A, b, G):
    grp = ThreadGroup(G)
    shards = []
    for q in range(G):
        j0, j1 = column_range(A.shape[0], q, G)
        P = Problem(np.ascontiguousarray(A[j0:j1]), b)
        shards.append((P, j0, j1))

    def attach(q):
        return lambda: shards[q][0].set_comm(grp.member(q), q, G)

    run_threads([attach(q) for q in range(G)], grp)
    return grp, shards


def sharded_solve(grp, shards, l1, l2, sigma0, tol, x0=None, x0_mask=None):
    def one(q):
        P, j0, j1 = shards[q]
        xs = None if x0 is None or (x0_mask is not None and not x0_mask[q]) else x0[j0:j1]
        return lambda: P.solve(l1, l2, sigma0, tol, x0=xs)

    res = run_threads([one(q) for q in range(len(shards))], grp)
    x = np.concatenate([r[0] for r in res])
    return x, [r[1] for r in res]


@pytest.mark.parametrize("name,n,G", [("cfg2", 20_000, 2), ("cfg3", 30_000, 3), ("cfg1", None, 2)])
def test_sharded_matches_single_and_oracle(name, n, G):
    cfg = synth.CONFIGS[name] if n is None else synth.scaled(synth.CONFIGS[name], n=n)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    lm1 = float(np.max(np.abs(oracle.aty(A, b))))
    lm = lm1 / cfg.alpha
    grp, shards = make_shards(A, b, G)
    try:
        for P, _, _ in shards:
            assert P.lambda_max_l1 == pytest.approx(lm1, rel=1e-13)  # global max after set_comm
        with Problem(A, b) as F:
            F.set_option("graph", 0)
            for c in (0.9, 0.3, 0.05):
                l1, l2 = c * cfg.alpha * lm, c * (1 - cfg.alpha) * lm
                xs, sts = sharded_solve(grp, shards, l1, l2, cfg.sigma0, cfg.tol)
                xf, sf = F.solve(l1, l2, cfg.sigma0, cfg.tol)
                xc, _, sc, _ = oracle.solve(A, b, l1, l2, sigma0=cfg.sigma0, tol=cfg.tol)
                s0 = sts[0]
                for s in sts[1:]:  # identical decisions on every shard
                    for k in ("status", "outer_iters", "newton_iters", "backtracks", "branch_steps", "active",
                              "res_kkt1", "res_kkt3", "primal_obj", "dual_obj"):
                        assert s[k] == s0[k], (k, s[k], s0[k])
                assert s0["status"] == 0 and sc["status"] == 0
                Fs = oracle.primal_obj(A, b, xs, l1, l2)
                Fc = oracle.primal_obj(A, b, xc, l1, l2)
                assert solution_parity(xs, xc, Fs, Fc)["ok"], (c, s0, sc)
                assert s0["outer_iters"] == sc["outer_iters"]
                assert abs(s0["newton_iters"] - sc["newton_iters"]) <= 1
                assert s0["active"] == int(np.count_nonzero(xs))
                assert s0["primal_obj"] == pytest.approx(Fs, rel=1e-12)
                assert np.max(np.abs(xs - xf)) <= 1e-7 * max(np.max(np.abs(xf)), 1e-300)
    finally:
        for P, _, _ in shards:
            P.close()


def test_sharded_warm_start_and_branches():
    cfg = synth.scaled(synth.CONFIGS["cfg2"], n=24_000)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    lm = float(np.max(np.abs(oracle.aty(A, b)))) / cfg.alpha
    G = 3
    grp, shards = make_shards(A, b, G)
    try:
        x = None
        seen = np.zeros(3, dtype=int)
        for c in (0.5, 0.3, 0.1):  # warm-started path
            l1, l2 = c * cfg.alpha * lm, c * (1 - cfg.alpha) * lm
            xprev = x
            x, sts = sharded_solve(grp, shards, l1, l2, cfg.sigma0, cfg.tol, x0=xprev)
            seen += np.array(sts[0]["branch_steps"][:3])
            xc, _, sc, _ = oracle.solve(A, b, l1, l2, sigma0=cfg.sigma0, tol=cfg.tol, x0=xprev)  # same warm start
            assert sts[0]["outer_iters"] == sc["outer_iters"] and abs(sts[0]["newton_iters"] - sc["newton_iters"]) <= 1
            assert solution_parity(x, xc, oracle.primal_obj(A, b, x, l1, l2), oracle.primal_obj(A, b, xc, l1, l2))["ok"]
        assert seen[1] > 0 and seen[2] > 0  # gathered-column SMW and summed-Gram m × m steps both ran
        # x0 on one shard only: the others count as zero (still a warm start)
        l1, l2 = 0.1 * cfg.alpha * lm, 0.1 * (1 - cfg.alpha) * lm
        xp, sts = sharded_solve(grp, shards, l1, l2, cfg.sigma0, 1e-8, x0=x, x0_mask=[True, False, False])
        j1 = column_range(cfg.n, 0, G)[1]
        x0_eff = np.concatenate([x[:j1], np.zeros(cfg.n - j1)])
        xc, _, sc, _ = oracle.solve(A, b, l1, l2, sigma0=cfg.sigma0, tol=1e-8, x0=x0_eff)
        assert sts[0]["status"] == 0
        assert solution_parity(xp, xc, oracle.primal_obj(A, b, xp, l1, l2), oracle.primal_obj(A, b, xc, l1, l2))["ok"]
        # hooks that need the whole matrix are refused on a sharded handle
        with pytest.raises(SsnalError):
            shards[0][0].model_select(l2)
    finally:
        for P, _, _ in shards:
            P.close()


def test_sharded_genotype_handles():
    """Packed 2-bit genotype shards (§8(f4) storage) exchange like fp64 ones: the gathered active
    columns and the summed Grams are decoded through the column accessor."""
    m, n, G = 300, 9000, 2
    cfg = synth.Config("gs", m, n, synth.GENO_STD, 10, 0.1, 0.3, 1.0, 0.5, (0.3,), 19)
    codes, tab = synth.geno_codes(cfg)
    A = synth.decode_geno(codes, tab, m)
    b, _ = synth.response(cfg)
    lm = float(np.max(np.abs(oracle.aty(A, b)))) / cfg.alpha
    grp = ThreadGroup(G)
    shards = []
    for q in range(G):
        j0, j1 = column_range(n, q, G)
        shards.append((Problem.from_geno(np.ascontiguousarray(codes[j0:j1]), np.ascontiguousarray(tab[j0:j1]), b),
                       j0, j1))
    try:
        run_threads([(lambda q=q: shards[q][0].set_comm(grp.member(q), q, G)) for q in range(G)], grp)
        for c in (0.3, 0.05):
            l1, l2 = c * cfg.alpha * lm, c * (1 - cfg.alpha) * lm
            xs, sts = sharded_solve(grp, shards, l1, l2, cfg.sigma0, cfg.tol)
            xc, _, sc, _ = oracle.solve(A, b, l1, l2, sigma0=cfg.sigma0, tol=cfg.tol)
            assert sts[0]["status"] == 0 and sts[0]["outer_iters"] == sc["outer_iters"]
            assert solution_parity(xs, xc, oracle.primal_obj(A, b, xs, l1, l2), oracle.primal_obj(A, b, xc, l1, l2))["ok"]
    finally:
        for P, _, _ in shards:
            P.close()
