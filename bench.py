#!/usr/bin/env python3
"""Benchmark of the SsNAL-EN hot path on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config cfg5|cfg1|cfg2|cfg3|cfg4] [--geno] [--sweep] [--select]

One "step" is one full time-to-solution of the workload at KKT tolerance 1e-6 — every §8(a) row of
SURVEY.md (K1 passes, re-thresholds, Newton systems, line searches, outer updates).  The default is
cfg5 (BASELINE configs[4], the "HBM-bound stress" case the metric's K1 target is stated on:
m = 500, n = 1e7, 40 GB of A, cold solves at c = 0.5 and 0.1); --config cfg2 times the 10-point
warm-started path of configs[1] (σ carried from point to point, reading R38).  Inputs are synthetic
(synth/), generated directly in HBM; A is larger than the 126 MB L2, so no flush is needed.

The JSON line carries: value (device-timed seconds per step, max over ranks) with per-step median and
mean ± se, e2e (the same workload through the host-memory C-ABI: ssnal_en_create from pinned HOST
buffers + the solves + x D2H inside the timed region), the roofline of the dominant kernel (K1:
algorithmic bytes per launch / mean launch time measured during the timed steps), cpu_baseline (the
oracle on this host's cores, warmed, in a clean subprocess; rank 0 only) and the §8(d) parity block of
the timed step's solutions against the oracle's, clocks sampled during the timed region, gpu_launches.

--impl reference: the base contract's reference arm is, for this paper-only tier, the CPU oracle
(oracle/), timed on the host cores with the same --steps/--warmup on a bounded column sample of the
same workload, scaled to seconds per workload (rank 0 only).
Multi-GPU (torchrun): by default each rank solves its own replica (value = max over ranks,
scaling "weak"); with --shard the ranks split the columns of one problem and
exchange the cross-column sums by NCCL all-reduce (scaling "strong").
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "time-to-solution (s) at KKT 1e-6; fused A^T·y kernel GB/s vs B200 HBM peak"


def _read_ceiling():
    """The best plain READ stream measured on this pool's B200s by tools/probes/read_probe (committed
    under profiles/): context for K1, which reads 8mn bytes and writes 8n; the roofline denominator stays
    the driver's copy rate."""
    p = os.path.join(ROOT, "profiles", "r2_read_ceiling_probe.jsonl")
    if not os.path.exists(p):
        return None
    best = 0.0
    for line in open(p):
        try:
            best = max(best, float(json.loads(line).get("GBps", 0.0)))
        except (ValueError, AttributeError):
            pass
    return best or None


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if "Active" in s[2 + i]
                          and not s[2 + i].startswith("Not")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def lambdas(cfg, lmax_l1, c):
    lmax = lmax_l1 / cfg.alpha
    return c * cfg.alpha * lmax, c * (1 - cfg.alpha) * lmax


def max_over_ranks(v: float, device: str = "cuda") -> float:
    """Max of a per-rank float over the process group (identity without one).  Works with
    NCCL (device='cuda') and gloo (device='cpu')."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(v)
    t = torch.tensor([float(v)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def k1_bytes(m, n, geno=False):
    """Algorithmic bytes of one fused K1 launch: A once (8mn fp64, or packed codes n·stride + 24n
    tables for the §8(f4) genotype storage), x read + w write (16n), y (8m)."""
    a = n * synth.geno_stride(m) + 24 * n if geno else 8 * m * n
    return a + 16 * n + 8 * m


def small_roofline(m, n, sts, dev_s, peak, peak_src):
    """Single-launch small-problem path (k_small_cl: one 16-CTA cluster, A resident in distributed
    shared memory; m ≤ 64, n ≤ 1024): no K1 launches; the whole solve is one latency-bound kernel.
    Reported: the effective A-pass bandwidth of the solve (passes × 8mn bytes / device time) against
    the HBM peak, for context only."""
    passes = sum(s["aty_passes"] for s in sts)
    achieved = passes * 8.0 * m * n / max(dev_s, 1e-30) / 1e9
    return {"bound": "latency", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": None, "peak_source": peak_src, "kernel": "k_small_cl",
            "bytes_per_launch": passes * 8 * m * n, "launches": len(sts), "mean_launch_us": dev_s / max(len(sts), 1) * 1e6,
            "share_of_step": 1.0,
            "note": "m <= 64, n <= 1024: Algorithm 1 in one launch of one 16-CTA cluster (A resident in distributed "
                    "shared memory); latency-bound (pivot chains, cluster barriers), not an HBM stream"}


def geno_roofline(m, n, k1_avg, k1_gbs, hbm_peak, traffic):
    """K1g (packed genotype codes) moves 32x fewer bytes than K1; its bucket sums run
    on the INT8 tensor cores (mma.sync m16n8k32 u8), and the per-element work that remains is
    expanding each 2-bit code into its two 0/1 bit planes for the MMA operand: ≥ 2 issued
    instructions per element (byte extract + 3-op spread per 4 elements and plane), so the bound is
    instruction issue — peak = 128 thread-instructions/clk/SM / 2 × 148 SMs × 1.965 GHz elements/s.
    The HBM view (algorithmic bytes / time vs the measured copy peak) is reported beside it."""
    peak_el = 128 / 2 * 148 * 1.965e9 / 1e9  # Gelem/s
    ach = m * n / k1_avg / 1e9 if k1_avg else None
    return {"bound": "alu", "achieved": ach, "peak": peak_el, "unit": "Gelem/s",
            "frac": (ach / peak_el) if ach else None, "traffic": traffic,
            "peak_source": "derived: issue bound of the 2-bit -> bit-plane expansion (2 instr/element at "
                           "128 thread-instr/clk/SM, 148 SMs, 1.965 GHz)",
            "hbm_view": {"achieved_GBps": k1_gbs, "peak_GBps": hbm_peak, "frac": (k1_gbs / hbm_peak) if k1_gbs else None}}


def run_step(P, cfg, lm, x_all):
    """One step: the workload's solves on device buffers (x_all: npts × n, row i = point i's x).
    Returns (device_s, launches, stats list).  A warm-started path goes through the library's path call
    (ssnal_en_solve_path_device: every point enqueued before one synchronisation, σ carried from point
    to point — reading R38); independent solves (cfg3-5) are cold solves, one per c."""
    if cfg.path:
        ls = [lambdas(cfg, lm, c) for c in cfg.cs]
        stats = P.solve_path_device([a for a, _ in ls], [b for _, b in ls], cfg.sigma0, cfg.tol, 0, x_all.data_ptr())
        return sum(s["time_device_s"] for s in stats), sum(s["kernel_launches"] for s in stats), stats
    total_dev, launches, stats = 0.0, 0, []
    for i, c in enumerate(cfg.cs):
        l1, l2 = lambdas(cfg, lm, c)
        st = P.solve_device(l1, l2, cfg.sigma0, cfg.tol, 0, x_all[i].data_ptr())
        total_dev += st["time_device_s"]
        launches += st["kernel_launches"]
        stats.append(st)
    return total_dev, launches, stats


def host_solve_workload(Q, cfg, lm):
    """The same workload through the host-memory C-ABI call ssnal_en_solve (x0 up, x down per solve).
    Returns (h2d bytes of the solves, d2h bytes)."""
    x_prev, sig, h2d, d2h = None, cfg.sigma0, 0, 0
    for i, c in enumerate(cfg.cs):
        l1, l2 = lambdas(cfg, lm, c)
        x0 = x_prev if (cfg.path and i > 0) else None
        Q.set_option("warm_dual", 1 if (cfg.path and i > 0) else 0)  # R39, as the path call does
        x_prev, st = Q.solve(l1, l2, sig, cfg.tol, x0=x0)
        if cfg.path:
            sig = st["sigma_final"]  # R38, as the path call does
        h2d += 8 * cfg.n if x0 is not None else 0
        d2h += 8 * cfg.n
    return h2d, d2h


def _host_room(bytes_per_rank, world):
    """Whether every local rank can pin its own host copy of A for the e2e leg (25% headroom)."""
    try:
        import psutil

        return psutil.virtual_memory().available > 1.25 * bytes_per_rank * world
    except Exception:
        return world == 1


def _host_room_all(bytes_per_rank, world):
    """_host_room decided jointly (every rank skips or runs the e2e leg: it contains collectives)."""
    ok = _host_room(bytes_per_rank, world)
    return ok if world == 1 else max_over_ranks(0.0 if ok else 1.0) == 0.0


def step_summary(ts):
    """median and mean ± standard error of per-step device times (SURVEY §8(d) timing protocol)."""
    ts = list(ts)
    mean = statistics.fmean(ts)
    se = statistics.stdev(ts) / len(ts) ** 0.5 if len(ts) > 1 else 0.0
    return {"median_s": statistics.median(ts), "mean_s": mean, "se_s": se, "n": len(ts)}


def bench_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2006_03970_b200 import Problem

    torch.cuda.set_device(local_rank)
    cfg = synth.CONFIGS[args.config]
    m, n = cfg.m, cfg.n
    stream = torch.cuda.current_stream()
    b_host, _ = synth.response(cfg)
    db = torch.from_numpy(b_host).cuda()
    dA = None
    if args.geno:  # §8(f4): A as packed 2-bit genotype codes + per-column tables
        if cfg.kind != synth.GENO_STD:
            raise SystemExit("--geno needs a genotype config (cfg4)")
        stride = synth.geno_stride(m)
        dcodes = torch.empty((n, stride), dtype=torch.uint8, device="cuda")
        dtab = torch.empty((n, 3), dtype=torch.float64, device="cuda")
        synth.fill_device_geno(cfg, dcodes.data_ptr(), dtab.data_ptr(), stream.cuda_stream)
        torch.cuda.synchronize()
        P = Problem.from_geno_device(dcodes.data_ptr(), stride, dtab.data_ptr(), db.data_ptr(), m, n,
                                     stream.cuda_stream, keep=(dcodes, dtab, db))
    elif args.shard:  # §8(f3): this rank owns columns [j0, j1); cross-column sums over the ranks
        from paper_2006_03970_b200.shard import attach_peers, column_range, torch_allreduce

        j0, j1 = column_range(cfg.n, rank, world)
        n = j1 - j0
        dA = torch.empty((n, m), dtype=torch.float64, device="cuda")
        synth.fill_device(cfg, dA.data_ptr(), stream.cuda_stream, j0, j1)
        torch.cuda.synchronize()
        P = Problem.from_device(dA.data_ptr(), db.data_ptr(), m, n, stream.cuda_stream, keep=(dA, db))
        if args.shard_comm == "peer":  # device-resident exchanges over peer memory (CUDA IPC, NVLink)
            attach_peers(P)
        else:  # a host callback per exchange: NCCL all-reduce (host-driven control)
            P.set_comm(torch_allreduce(), rank, world)
    else:
        dA = torch.empty((n, m), dtype=torch.float64, device="cuda")
        synth.fill_device(cfg, dA.data_ptr(), stream.cuda_stream)
        torch.cuda.synchronize()
        P = Problem.from_device(dA.data_ptr(), db.data_ptr(), m, n, stream.cuda_stream, keep=(dA, db))
    P.set_option("graph", 1 if args.control == "graph" else 0)
    P.set_option("cg_ratio", args.cg_ratio)
    for kv in args.opt:  # library options for A/B runs (recorded in config)
        k, v = kv.split("=")
        P.set_option(k, float(v))
    lm = P.lambda_max_l1
    x_all = torch.zeros((len(cfg.cs), n), dtype=torch.float64, device="cuda")

    for _ in range(args.warmup):
        run_step(P, cfg, lm, x_all)
    torch.cuda.synchronize()

    # ---- timed region: K steps, K1 launch times on the handle's stream ----
    P.set_option("time_k1", 1)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    k1_time = 0.0
    k1_launches = 0
    launches = 0
    dev_sum = 0.0
    last_stats = None
    reuses0 = P.info("atb_reuses")
    with ClockSampler(local_rank) as clk:
        evs[0].record(stream)
        for k in range(args.steps):
            d, L, sts = run_step(P, cfg, lm, x_all)
            evs[k + 1].record(stream)
            dev_sum += d
            launches += L
            k1_time += sum(s["k1_time_s"] for s in sts)
            k1_launches += sum(s["k1_launches"] for s in sts)
            last_stats = sts
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    P.set_option("time_k1", 0)
    atb_reuses = (P.info("atb_reuses") - reuses0) / max(args.steps, 1)
    per_step = [evs[k].elapsed_time(evs[k + 1]) * 1e-3 for k in range(args.steps)]
    elapsed = sum(per_step)
    t_step = max_over_ranks(elapsed / args.steps)
    x_gpu = x_all.cpu().numpy()  # the last timed step's solutions (parity block)

    # K1 at a probe point for the parity block's Aᵀy error (R21): same y as the oracle leg
    w_probe = None
    if rank == 0 and world == 1 and not args.no_cpu and not args.shard:
        y = torch.from_numpy(synth.normals(cfg.seed, 12, m)).cuda()
        xz = torch.zeros(n, dtype=torch.float64, device="cuda")
        w = torch.empty(n, dtype=torch.float64, device="cuda")
        J = torch.empty(n, dtype=torch.int32, device="cuda")
        PJ = torch.empty(n, dtype=torch.float64, device="cuda")
        P.aty_fused(y.data_ptr(), xz.data_ptr(), 1.0, 1e300, 0.1, w.data_ptr(), J.data_ptr(), PJ.data_ptr())
        w_probe = w.cpu().numpy()
        del y, xz, w, J, PJ

    # ---- e2e: the public host-memory C-ABI with HOST buffers; per step: ssnal_en_create (H2D of A, b,
    # validation, λmax pass), the workload's solves through ssnal_en_solve (x0 H2D, x D2H), destroy ----
    e2e = None
    if not args.no_e2e and args.geno:
        codes_h, tab_h = synth.geno_codes(cfg)
        e2e_times = []
        for it in range(max(1, min(args.steps, 3)) + 1):
            t0 = time.perf_counter()
            Q = Problem.from_geno(codes_h, tab_h, b_host)
            Q.set_option("graph", 1 if args.control == "graph" else 0)
            h2d, d2h = host_solve_workload(Q, cfg, Q.lambda_max_l1)
            Q.close()
            if it > 0:
                e2e_times.append(time.perf_counter() - t0)
        e2e = {"value": max_over_ranks(statistics.median(e2e_times)), "unit": "s",
               "h2d_bytes_per_step": int(codes_h.nbytes + tab_h.nbytes + 8 * m + h2d),
               "d2h_bytes_per_step": d2h, "steps": len(e2e_times),
               "includes": "create (H2D codes + tables + b, validation, lambda_max pass) + solves + D2H x + destroy"}
        del codes_h, tab_h
    elif not args.no_e2e and not args.shard and not _host_room_all(8 * m * n, world):
        e2e = {"value": None, "unit": "s", "skipped": f"host RAM: {world} rank(s) x {8 * m * n / 1e9:.0f} GB of pinned A "
                                                     "would not fit (psutil available memory)"}
    elif not args.no_e2e and not args.shard:
        A_host = torch.empty((n, m), dtype=torch.float64, pin_memory=True)
        A_host.copy_(dA)  # the same bytes as the device generator wrote (pinned host memory)
        A_np = A_host.numpy()
        e2e_times = []
        for it in range(max(1, min(args.steps, 3)) + 1):
            t0 = time.perf_counter()
            Q = Problem(A_np, b_host)
            Q.set_option("graph", 1 if args.control == "graph" else 0)
            Q.set_option("cg_ratio", args.cg_ratio)
            h2d, d2h = host_solve_workload(Q, cfg, Q.lambda_max_l1)
            Q.close()
            if it > 0:  # the first iteration is the e2e warm-up
                e2e_times.append(time.perf_counter() - t0)
        del A_np, A_host
        e2e = {"value": max_over_ranks(statistics.median(e2e_times)), "unit": "s",
               "h2d_bytes_per_step": 8 * m * n + 8 * m + h2d, "d2h_bytes_per_step": d2h,
               "steps": len(e2e_times),
               "includes": "ssnal_en_create (H2D of A and b from pinned host memory, validation, lambda_max pass)"
                           " + the workload's ssnal_en_solve calls (x0 H2D, x D2H) + destroy"}

    peak, peak_src = _peaks()
    k1_avg = k1_time / max(k1_launches, 1)
    k1_gbs = k1_bytes(m, n, args.geno) / k1_avg / 1e9 if k1_launches else None
    traffic = None
    tp = os.path.join(ROOT, "profiles", "k1_traffic.json")
    if os.path.exists(tp):
        try:
            tj = json.load(open(tp))
            traffic = tj.get(args.config + ("_geno" if args.geno else ""))
        except Exception:
            traffic = None
    res = {
        "metric": METRIC,
        "value": t_step,
        "unit": "s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t_step * 1e3,
        "higher_is_better": False,
        "scaling": "strong" if args.shard else "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (synth/, seeded; generated in HBM)",
        "config": {"workload": f"{cfg.name}: m={m} n={cfg.n} " + ("warm-started path c=" + ",".join(f"{c:.3g}" for c in cfg.cs)
                                                              if cfg.path else "cold solves c=" + ",".join(str(c) for c in cfg.cs)),
                   "m": m, "n": cfg.n, "alpha": cfg.alpha, "tol": cfg.tol, "sigma0": cfg.sigma0,
                   "l2_policy": f"A = {8 * m * n / 1e6:.0f} MB > 126 MB L2 (no flush needed)",
                   "parallelism": ((f"column-sharded x{world}: rank q owns n/{world} columns; per-evaluation "
                                    "partials and the Newton-system exchange (SURVEY 8(f3)) "
                                    + ("as device kernels over peer memory (CUDA IPC regions, rank-ordered sums)"
                                       if args.shard_comm == "peer" else "by NCCL all-reduce host callbacks"))
                                   if args.shard else f"replicas x{world}"),
                   "control": ("device-resident, one CUDA graph per solve (nested conditional WHILE)"
                               if args.control == "graph" and (not args.shard or args.shard_comm == "peer")
                               else "host-driven (per-evaluation readback)"),
                   "storage": ("packed 2-bit genotype codes + per-column tables (SURVEY 8(f4))" if args.geno
                               else "fp64 column-major"),
                   "path_sigma": "carried from point to point (reading R38, P:411)" if cfg.path else None,
                   "path_dual": ("each point after the first starts from the previous point's final y, w = A^T y "
                                 "(reading R39, P:236-246 + P:409-411): no A^T pass for the warm start")
                                if cfg.path else None,
                   "reuse_atb": ((f"on (reading R40): in {atb_reuses:g} of the step's cold solves K1 was allowed to serve a "
                                  "trial at y == -b (bitwise; the first Newton steps after x0 = 0, while J is empty: "
                                  "d = -(y + b)) from the A^T b kept by create's lambda_max pass instead of streaming A; "
                                  "bitwise the streamed result (tests/test_gpu_reuse.py); with the grad-psi rows gathered while "
                                  "#{|A^T b|_i > lambda1} <= 0.3 n, psi-only above (Armijo rejects s = 1 there; if it accepts, the "
                                  "trial is redone streamed); designs >= 2 GB; such launches are not counted in roofline.launches; "
                                  "--opt reuse_atb=0 times without it")
                                 if P.info("reuse_atb") == 1 else "off"),
                   "newton_strategy": ("exact (Eq. 18/19); CG when min(m, r) > 1e4 (P:379)" if args.cg_ratio == 0
                                       else f"CG (K6) when r > {args.cg_ratio:g} m, else exact (Eq. 18/19)")},
        "step_times": step_summary(per_step),
        "roofline": small_roofline(m, n, last_stats, dev_sum / max(args.steps, 1), peak, peak_src) if k1_launches == 0 and
                    not args.geno else {**({"bound": "hbm", "achieved": k1_gbs, "peak": peak, "unit": "GB/s",
                         "frac": (k1_gbs / peak) if k1_gbs else None, "traffic": traffic, "peak_source": peak_src,
                         "frac_of_nominal_8TBps": (k1_gbs / 8000.0) if k1_gbs else None,
                         "read_ceiling_GBps": _read_ceiling(),
                         "frac_of_read_ceiling": (k1_gbs / _read_ceiling()) if (k1_gbs and _read_ceiling()) else None,
                         "note": "peak = the driver's measured copy rate (read+write bytes of a bf16 copy); a "
                                 "read-dominated stream can exceed it, so frac > 1 is possible; the nominal "
                                 "8 TB/s view is frac_of_nominal_8TBps (north-star target >= 0.70); read_ceiling_GBps "
                                 "is the best plain read stream of tools/probes/read_probe on this pool"}
                        if not args.geno else geno_roofline(m, n, k1_avg, k1_gbs, peak, traffic)),
                     "kernel": "k1g_aty_fused" if args.geno else "k1_aty_fused",
                     "bytes_per_launch": k1_bytes(m, n, args.geno), "launches": k1_launches,
                     "mean_launch_us": k1_avg * 1e6, "share_of_step": k1_time / max(elapsed, 1e-30),
                     "timing": "in-kernel %globaltimer stamps inside the graph (CUDA events cannot sit in "
                               "conditional bodies) + CUDA events on the handle's stream for the warm-start passes"},
        "e2e": e2e,
        "gpu_launches": launches // max(args.steps, 1),
        "solves_device_s_per_step": dev_sum / max(args.steps, 1),
        "clocks": clk.summary(),
        "iterations": [{"c": round(c, 4), "outer": s["outer_iters"], "newton": s["newton_iters"],
                        "passes": s["aty_passes"], "backtracks": s["backtracks"], "r": s["active"],
                        "branches": s["branch_steps"], "cg_iters": s["cg_iters"], "sigma_final": s["sigma_final"],
                        "res1": s["res_kkt1"], "res3": s["res_kkt3"], "gap": s["gap"]}
                       for c, s in zip(cfg.cs, last_stats)],
    }
    if args.shard:
        res["config"]["n_local"] = n
    if args.opt:
        res["config"]["options"] = dict(kv.split("=") for kv in args.opt)
    P.close()
    del dA, x_all
    torch.cuda.empty_cache()
    if rank == 0 and not args.no_cpu and world == 1 and not args.shard:
        cb, parity = cpu_baseline(cfg, args, x_gpu, w_probe, last_stats)
        res["cpu_baseline"] = cb
        res["parity"] = parity
    return res


def _cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def cpu_baseline(cfg, args, x_gpu, w_probe, gpu_stats):
    """The oracle (as it stands) on this host's cores, in a CLEAN subprocess (no torch, no CUDA): it
    generates A with synth's host generator, warms up with one Aᵀb pass (OpenMP threads up, A paged
    in), then times the workload once — the full config, the same solves as one GPU step.  It also
    returns the §8(d) parity block of the GPU's last timed step against its own solutions."""
    import tempfile

    tmp = tempfile.mkdtemp(prefix="ssnal_bench_")
    np.save(os.path.join(tmp, "x_gpu.npy"), x_gpu)
    if w_probe is not None:
        np.save(os.path.join(tmp, "w_gpu.npy"), w_probe)
    json.dump([{k: s[k] for k in ("outer_iters", "newton_iters", "active", "status")} for s in gpu_stats],
              open(os.path.join(tmp, "gpu_stats.json"), "w"))
    out = os.path.join(tmp, "cpu.json")
    env = dict(os.environ)
    threads = int(env.get("OMP_NUM_THREADS", os.cpu_count()))
    env["OMP_NUM_THREADS"] = str(threads)
    cmd = [sys.executable, os.path.abspath(__file__), "--cpu-leg", tmp, "--config", cfg.name]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True)
    if r.returncode != 0 or not os.path.exists(out):
        return {"value": None, "unit": "s", "cores": threads, "kind": "oracle",
                "error": (r.stderr or r.stdout)[-400:]}, None
    d = json.load(open(out))
    cb = d["cpu_baseline"]
    if cfg.name in ("cfg1", "cfg2", "cfg3") and threads > 1:
        # the oracle also at one thread for the configs where that stays bounded
        os.remove(os.path.join(tmp, "x_gpu.npy"))  # timing only, no second parity block
        env["OMP_NUM_THREADS"] = "1"
        r1 = subprocess.run(cmd, env=env, capture_output=True, text=True)
        if r1.returncode == 0 and os.path.exists(out):
            d1 = json.load(open(out))["cpu_baseline"]
            cb["one_thread"] = {"value": d1["value"], "threads": 1, "speedup_nproc": d1["value"] / cb["value"]}
    for f in os.listdir(tmp):
        os.remove(os.path.join(tmp, f))
    os.rmdir(tmp)
    return cb, d["parity"]


def cpu_leg(tmp, cfg_name):
    """Child process of cpu_baseline (no torch): oracle timing + parity block, written to tmp/cpu.json."""
    import oracle

    cfg = synth.CONFIGS[cfg_name]
    t_gen = time.perf_counter()
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    t_gen = time.perf_counter() - t_gen
    t0 = time.perf_counter()
    lm = oracle.lambda_max_l1(A, b)  # warm-up: one full Aᵀb pass
    t_warm = time.perf_counter() - t0
    ls = [lambdas(cfg, lm, c) for c in cfg.cs]
    t0 = time.perf_counter()
    if cfg.path:
        sols = oracle.solve_path_lambdas(A, b, ls, sigma0=cfg.sigma0, tol=cfg.tol)
    else:
        sols = [oracle.solve(A, b, l1, l2, sigma0=cfg.sigma0, tol=cfg.tol)[:3] for l1, l2 in ls]
    dt = time.perf_counter() - t0
    threads = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count()))
    cb = {"value": dt, "unit": "s", "cores": threads, "kind": "oracle",
          "sample": f"the full {cfg.name} workload ({len(ls)} solve(s){', warm-started path, sigma carried' if cfg.path else ''}),"
                    " one timed run after a warm-up A^T b pass; clean subprocess (no torch), OpenMP over columns",
          "threads": threads, "nproc": os.cpu_count(), "cpu_model": _cpu_model(),
          "generate_s": t_gen, "warmup_s": t_warm,
          "iterations": [{"outer": s["outer_iters"], "newton": s["newton_iters"], "r": s["active"]} for _, _, s in sols]}
    parity = None
    xg_path = os.path.join(tmp, "x_gpu.npy")
    if os.path.exists(xg_path):
        x_gpu = np.load(xg_path)
        gst = json.load(open(os.path.join(tmp, "gpu_stats.json")))
        pts = []
        for i, ((l1, l2), (xc, _, sc)) in enumerate(zip(ls, sols)):
            xg = x_gpu[i]
            Fg, Fc = oracle.primal_obj(A, b, xg, l1, l2), oracle.primal_obj(A, b, xc, l1, l2)
            xinf = float(np.max(np.abs(xc)))
            mask = np.maximum(np.abs(xg), np.abs(xc)) > 1e-8
            pts.append({"c": cfg.cs[i], "obj_rel": abs(Fg - Fc) / abs(Fc),
                        "xinf_rel": float(np.max(np.abs(xg - xc))) / max(xinf, 1e-300),
                        "sign_match": bool(np.array_equal(np.sign(xg[mask]), np.sign(xc[mask]))),
                        "J_equal": bool(np.array_equal(np.nonzero(xg)[0], np.nonzero(xc)[0])),
                        "outer": [gst[i]["outer_iters"], sc["outer_iters"]],
                        "newton": [gst[i]["newton_iters"], sc["newton_iters"]]})
        ok = all(p["obj_rel"] <= 1e-9 and p["xinf_rel"] <= 1e-6 and p["sign_match"] for p in pts)
        parity = {"points": pts, "ok": ok,
                  "tolerances": "objective 1e-9 rel, |dx|inf <= 1e-6 |x_cpu|inf, sign pattern on |x|>1e-8 (BASELINE "
                                "north star; R22); gpu/oracle = [gpu, oracle] counts"}
        wg_path = os.path.join(tmp, "w_gpu.npy")
        if os.path.exists(wg_path):  # K1 vs the oracle's Aᵀy at the probe y (reading R21)
            w_gpu = np.load(wg_path)
            y = synth.normals(cfg.seed, 12, cfg.m)
            w_cpu = oracle.aty(A, y)
            ny = float(np.linalg.norm(y))
            e1 = 0.0
            for j in range(0, cfg.n, 1 << 20):
                blk = A[j:j + (1 << 20)]
                cn = np.sqrt(np.einsum("ij,ij->i", blk, blk))
                e1 = max(e1, float(np.max(np.abs(w_gpu[j:j + len(blk)] - w_cpu[j:j + len(blk)]) / (cn * ny))))
            parity["aty_max_scaled_err"] = e1
            parity["aty_rel_l2_err"] = float(np.linalg.norm(w_gpu - w_cpu) / np.linalg.norm(w_cpu))
            parity["ok"] = parity["ok"] and e1 <= 1e-12
    json.dump({"cpu_baseline": cb, "parity": parity}, open(os.path.join(tmp, "cpu.json"), "w"))


def bench_reference(args, rank, world):
    """Reference arm for this tier: the CPU oracle (as it stands) on the host cores, rank 0 only, with
    the same --steps/--warmup as our arm.  Each step is a bounded sample of the workload: the same
    solves on the first n_s columns of the same design (synth, same generator and b), λmax of the
    sample; the step time is scaled by n / n_s to the metric's unit (seconds per full workload; the
    oracle's cost is linear in n: every Newton step is an O(mn) pass).  n_s = n for cfg1/cfg2/cfg4."""
    if rank != 0:
        return None
    import oracle

    cfg = synth.CONFIGS[args.config]
    frac = {"cfg3": 0.5, "cfg5": 0.2}.get(cfg.name, 1.0)
    ns = int(cfg.n * frac)
    A = synth.design(cfg, 0, ns)
    b, _ = synth.response(cfg)
    lm = oracle.lambda_max_l1(A, b)
    ls = [lambdas(cfg, lm, c) for c in cfg.cs]

    def step():
        if cfg.path:
            oracle.solve_path_lambdas(A, b, ls, sigma0=cfg.sigma0, tol=cfg.tol)
        else:
            for l1, l2 in ls:
                oracle.solve(A, b, l1, l2, sigma0=cfg.sigma0, tol=cfg.tol)

    for _ in range(args.warmup):
        step()
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        ts.append(time.perf_counter() - t0)
    scale = cfg.n / ns
    t = statistics.fmean(ts) * scale
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count()))
    sample = (f"full {cfg.name} workload per step" if ns == cfg.n else
              f"{cfg.name} workload on the first {ns} of {cfg.n} columns (same generator and b, its own lambda_max), "
              f"time x {scale:g}")
    return {"impl": "reference", "metric": METRIC, "value": t, "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (synth/, seeded)",
            "config": {"workload": f"{cfg.name}: m={cfg.m} n={cfg.n} " + ("warm-started path" if cfg.path else
                                   "cold solves c=" + ",".join(str(c) for c in cfg.cs)),
                       "m": cfg.m, "n": cfg.n, "sample_columns": ns},
            "step_times": step_summary([v * scale for v in ts]),
            "cpu_baseline": {"value": t, "unit": "s", "cores": cores, "kind": "oracle", "sample": sample,
                             "cpu_model": _cpu_model()},
            "e2e": {"value": t, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def bench_select(args):
    """the Table D.4 protocol on cfg2 — 100 log-spaced c from 1 to 0.1,
    warm-started, stopping at 100 active features, with ν / OLS de-biasing / GCV / e-BIC at
    every point.  GPU device time per path vs the oracle doing the same on the host."""
    import torch

    from paper_2006_03970_b200 import Problem
    from paper_2006_03970_b200.path import lambda_grid, solve_path

    cfg = synth.CONFIGS["cfg2"]
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    cs = lambda_grid(100)
    P = Problem(A, b)
    for _ in range(max(args.warmup, 1)):
        solve_path(P, cfg.alpha, cs, max_active=100)
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        pts, best = solve_path(P, cfg.alpha, cs, max_active=100)
        ts.append(time.perf_counter() - t0)
    lm_l1 = P.lambda_max_l1  # ‖Aᵀb‖∞ from the handle's own K1 pass (the CV grid is the full-data one)
    P.close()
    t_gpu = statistics.median(ts)
    res = {"metric": "lambda-path with model selection: time per path (s)", "value": t_gpu, "unit": "s",
           "higher_is_better": False, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "dtype": "f64",
           "data": "synthetic (synth/, seeded)",
           "config": {"workload": "cfg2 path: 100 log-spaced c in [0.1, 1], max 100 actives (Table D.4 protocol)",
                      "points": len(pts), "best_gcv": best["gcv"], "best_ebic": best["ebic"]}}
    if not args.no_cpu:
        import oracle

        lm = float(np.max(np.abs(oracle.aty(A, b)))) / cfg.alpha
        t0 = time.perf_counter()
        x = None
        for c in cs:
            l1, l2 = c * cfg.alpha * lm, c * (1 - cfg.alpha) * lm
            x, _, st, _ = oracle.solve(A, b, l1, l2, x0=x)
            oracle.model_select(A, b, x, l2)
            if st["active"] >= 100:
                break
        res["cpu_baseline"] = {"value": time.perf_counter() - t0, "unit": "s", "cores": os.cpu_count(),
                               "kind": "oracle", "sample": "the same path with the same criteria"}
    if args.cv > 0:  # k-fold CV along a 20-point grid (reading R35)
        from paper_2006_03970_b200.path import cv_path

        dA = torch.from_numpy(A).cuda()
        st = torch.cuda.current_stream()

        def make(rows):
            sub = dA[:, torch.from_numpy(rows).cuda()].contiguous()
            bs = torch.from_numpy(np.ascontiguousarray(b[rows])).cuda()
            return Problem.from_device(sub.data_ptr(), bs.data_ptr(), len(rows), cfg.n, st.cuda_stream,
                                       keep=(sub, bs))

        cs_cv = lambda_grid(20)
        cv_path(make, cfg.m, cfg.alpha, cs_cv, lm_l1, k=args.cv)  # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cv, best = cv_path(make, cfg.m, cfg.alpha, cs_cv, lm_l1, k=args.cv)
        torch.cuda.synchronize()
        res["cv"] = {"k": args.cv, "points": len(cs_cv), "seconds": time.perf_counter() - t0, "best": best,
                     "best_c": float(cs_cv[best])}
        if not args.no_cpu:
            import oracle

            t0 = time.perf_counter()
            cvc, bestc = oracle.cv_path(A, b, cfg.alpha, cs_cv, k=args.cv)
            res["cv"]["cpu_baseline"] = {"value": time.perf_counter() - t0, "unit": "s", "kind": "oracle",
                                         "best": bestc, "max_rel_diff": float(np.max(np.abs(cv - cvc) / cvc))}
    print(json.dumps(res), flush=True)


def sweep(args):
    """K1 bandwidth sweep: m = 500, n = 1e5 … 1e7, plus spot checks at m = 50 and m = 800
    (n = 1e6); y ~ N(0, I), x with 100 nonzeros ±U[1,2], σ = 1, λ1 at the (1 − 1e-4) quantile of |x − σAᵀy|
    (r ≈ 1e-4 n, the typical regime) and at the median (r ≈ n/2, the compaction worst case); median of
    --sweep-reps launches.  t_k1 = CUDA events around the K1 launch alone (option time_k1, get_info
    "k1_time_s"); t_call = the whole hook (K1 + the ordered concatenation + the ψ/∇ψ reduction + sync)."""
    import torch

    from paper_2006_03970_b200 import Problem

    peak, _ = _peaks()
    stream = torch.cuda.current_stream()
    cases = [(500, int(v)) for v in args.sweep_n.split(",")] + [(50, 1_000_000), (800, 1_000_000)]
    for m in sorted({mm for mm, _ in cases}):
        base = synth.scaled(synth.CONFIGS["cfg5"], m=m, n=max(nn for mm, nn in cases if mm == m))
        dA = torch.empty((base.n, m), dtype=torch.float64, device="cuda")
        synth.fill_device(base, dA.data_ptr(), stream.cuda_stream)
        torch.cuda.synchronize()
        for n in [nn for mm, nn in cases if mm == m]:
            b = torch.from_numpy(synth.normals(5, 11, m)).cuda()
            P = Problem.from_device(dA.data_ptr(), b.data_ptr(), m, n, stream.cuda_stream, keep=(dA, b))
            if args.k1_stages:
                P.set_option("k1_stages", args.k1_stages)
            y = torch.from_numpy(synth.normals(5, 12, m)).cuda()
            xh = np.zeros(n)
            k = min(100, n)
            idx = np.unique((synth.uniforms(5, 13, k) * n).astype(np.int64) % n)
            xh[idx] = np.where(synth.uniforms(5, 14, len(idx)) < 0.5, -1.0, 1.0) * (1.0 + synth.uniforms(5, 15, len(idx)))
            x = torch.from_numpy(xh).cuda()
            w = torch.empty(n, dtype=torch.float64, device="cuda")
            J = torch.empty(n, dtype=torch.int32, device="cuda")
            PJ = torch.empty(n, dtype=torch.float64, device="cuda")
            P.aty_fused(y.data_ptr(), x.data_ptr(), 1.0, 1e30, 0.1, w.data_ptr(), J.data_ptr(), PJ.data_ptr())
            t_abs = (x - w).abs()[: min(n, 16_000_000)].float()  # |x − σw| with σ = 1
            q = float(torch.quantile(t_abs, 1 - 1e-4).item()) if n > 1 else 0.0
            for lab, l1 in (("r~1e-4n", q), ("r~n/2", float(t_abs.median().item()))):
                ts = []
                for it in range(args.sweep_reps + 3):
                    if it == 3:
                        P.set_option("time_k1", 1)  # resets the K1 accumulators after the warm-ups
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    r, _ = P.aty_fused(y.data_ptr(), x.data_ptr(), 1.0, l1, 0.1, w.data_ptr(), J.data_ptr(),
                                       PJ.data_ptr())
                    e1.record(stream)
                    torch.cuda.synchronize()
                    if it >= 3:
                        ts.append(e0.elapsed_time(e1) * 1e-3)
                t_call = statistics.median(ts)
                t_k1 = P.info("k1_time_s") / max(P.info("k1_launches"), 1)
                P.set_option("time_k1", 0)
                gbs = k1_bytes(m, n) / t_k1 / 1e9
                print(json.dumps({"sweep": "k1", "m": m, "n": n, "case": lab, "r": r, "k1_stages": P.info("k1_stages"),
                                  "t_k1_us": t_k1 * 1e6,
                                  "t_call_us": t_call * 1e6, "GBps": gbs, "frac_of_measured": gbs / peak,
                                  "pct_of_8TBps": gbs / 8000}), flush=True)
            P.close()
        del dA
        torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg5", choices=list(synth.CONFIGS))
    ap.add_argument("--cpu-leg", default=None, help=argparse.SUPPRESS)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--geno", action="store_true",
                    help="cfg4 from packed 2-bit genotype codes (SURVEY 8(f4)) instead of fp64")
    ap.add_argument("--cg-ratio", type=float, default=0.0,
                    help="Newton strategy: CG when r > ratio*m (0: the paper's rule, min(m, r) > 1e4)")
    ap.add_argument("--control", default="graph", choices=["graph", "host"],
                    help="graph: Algorithm 1 control on the device in one CUDA graph; host: CPU decisions")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer e2e leg (40 GB configs)")
    ap.add_argument("--sweep", action="store_true", help="K1 bandwidth sweep instead of the TTS bench")
    ap.add_argument("--select", action="store_true", help="lambda path with model selection (SURVEY 8(f1))")
    ap.add_argument("--cv", type=int, default=0, help="with --select: k-fold cross-validation over a 20-point grid")
    ap.add_argument("--shard", action="store_true",
                    help="column-sharded solve across the ranks (SURVEY 8(f3)) instead of replicas")
    ap.add_argument("--shard-comm", default="peer", choices=["peer", "nccl"],
                    help="with --shard: device-resident exchanges over peer memory (default) or NCCL host callbacks")
    ap.add_argument("--sweep-n", default="100000,200000,500000,1000000,2000000,5000000,10000000")
    ap.add_argument("--sweep-reps", type=int, default=50)
    ap.add_argument("--k1-stages", type=int, default=0, help="with --sweep: K1 ring depth (0 = the library default)")
    ap.add_argument("--opt", action="append", default=[], help="library option key=value for the run (repeatable)")
    args = ap.parse_args()
    if args.cpu_leg:
        cpu_leg(args.cpu_leg, args.config)
        return
    if args.warmup < 3 and args.impl == "ours" and not args.sweep:
        args.warmup = 3  # contract: W ≥ 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook (tools/, never used for a reported number): run the multi-rank code path with every
    # rank on device 0 and a gloo group, on a box with one GPU
    if os.environ.get("BENCH_TEST_ONE_DEVICE") == "1":
        local_rank = 0
        if world > 1:  # ranks sharing one GPU must not spin on one another: host-callback exchanges
            args.shard_comm = "nccl"

    if args.impl == "reference":
        res = bench_reference(args, rank, world)
        if res is not None:
            print(json.dumps(res), flush=True)
        return

    if args.sweep:
        sweep(args)
        return
    if args.select:
        bench_select(args)
        return

    import torch.distributed as dist

    if world > 1 or args.shard:
        import torch

        torch.cuda.set_device(local_rank)
        if world > 1:
            dist.init_process_group("gloo" if os.environ.get("BENCH_TEST_ONE_DEVICE") == "1" else "nccl")
        else:  # a one-rank NCCL group, so the sharded path runs its real all-reduces
            import socket

            with socket.socket() as so:
                so.bind(("127.0.0.1", 0))
                port = so.getsockname()[1]
            dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    res = bench_ours(args, rank, world, local_rank)
    if rank == 0:
        print(json.dumps(res), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
