// k_ctl.cuh — device-resident control of Algorithm 1 (graph mode).
//
// In graph mode the whole solve is one CUDA graph: nested conditional WHILE nodes
//   outer (k)  : σ-scalars, EVAL at (y, x), inner loop, multiplier update, σ ← 5σ
//   inner (j)  : Newton direction, trial K1 at y + d, Armijo test, backtrack loop, accept
//   backtrack  : y + s d, K1e from w + s (w1 − w), Armijo test
// The decisions that the host-driven mode takes on the CPU (inner stop, branch on r, Armijo,
// KKT stop, σ update) are taken here by single-thread control kernels reading the EvalOut
// records in device memory, with the same IEEE operations in the same order (explicit _rn
// intrinsics, no contraction) — both modes give bitwise-identical iterates and stats.
// Buffers have fixed roles: index 0 = current point, 1 = trial, w[2] = backtrack; accepting a
// step copies trial → current on the device (k_accept).
#pragma once
#include "common.cuh"
#include "k_aty.cuh"
#include "k_newton.cuh"
#include "k_cg.cuh"

namespace ssn {

struct DevCtl {
  // per-solve settings (host-written before the graph launch)
  double l1, l2, tol, sigma, sigma_factor, sigma_max, mu, beta;
  double cg_ratio, cg_threshold;  // Newton strategy (R32)
  double nb;                      // ‖b‖ (res1 denominator, Eq. (15))
  double jitter;                  // factor retry scale (R36); 0 = no retry
  int max_outer, max_inner, max_bt;
  int reuse_mode;  // R40 (the reuse graph): how its trial K1 serves y == −b — 1 with the ∇ψ rows, 2 ψ only (K1Params::rmode)
  // state
  Scal sc;           // σ-dependent scalars of the current outer iteration
  double kinv;       // 1/κ
  double s, gd;      // Armijo step length and gᵀd of the current direction
  int k, j, nbt, need_grad;
  int converged, numeric, numeric_kind, stalled;
  int retry, skip;   // retry: this step's factor failed once; skip: redo the step (no accept)
  int inject;        // test hook: treat the next `inject` factorisations as failed
  int inner_tol_mode;  // 0: tol_in = tol (R6); 1: tol_in = max(tol, 0.1 res3 at the outer start) (R37)
  double tol_in;     // inner stop of the current outer iteration
  DirGeo geo;        // direction geometry for the current r
  // statistics (same meaning as ssnal_en_stats)
  int outer_iters, newton_iters, psi_evals, backtracks, aty_passes, branch_steps[4], cg_iters;
  int seg_outer, seg_inner, seg_bt, seg_grad;  // segment executions (kernel-launch accounting)
  double res1, res3, sigma_final;
  long long numeric_r;
  unsigned long long k1_ns;  // Σ K1 durations from the in-kernel globaltimer stamps
  int k1_cnt, jitter_retries;
  unsigned long long tstamp[2];
  int gmiss;  // R40: the last trial K1 was served ψ-only — its ∇ψ rows are missing
  int redo;   // R40: Armijo accepted s = 1 on such a trial: the redo nodes stream the pass and decide again
};

constexpr double kEpsDev = 2.220446049250313e-16;

SSN_DEV Scal make_scal_dev(double sigma, double l1, double l2) {
  Scal s;
  s.sigma = sigma;
  s.l1 = l1;
  s.l2 = l2;
  s.thr = __dmul_rn(sigma, l1);
  s.den = __dadd_rn(1.0, __dmul_rn(sigma, l2));
  s.cpsi = __ddiv_rn(__dadd_rn(1.0, __dmul_rn(sigma, l2)), __dmul_rn(2.0, sigma));
  s.kappa = __ddiv_rn(sigma, __dadd_rn(1.0, __dmul_rn(sigma, l2)));
  return s;
}

// Armijo, Eq. (13) with μ and the roundoff guard of reading R29:
//   ψ(y + s d) − ψ(y) ≤ μ s gᵀd + 10 ε |ψ|
SSN_DEV bool armijo_ok(const DevCtl* C, double psi_t, double psi0, double psimag0) {
  const double lhs = __dsub_rn(psi_t, psi0);
  const double rhs = __dadd_rn(__dmul_rn(__dmul_rn(C->mu, C->s), C->gd), __dmul_rn(__dmul_rn(10.0, kEpsDev), psimag0));
  return lhs <= rhs;
}

// After a test at step s: stop (accept s), stop stalled (R30), or halve (R5) and go on.
SSN_DEV int bt_next(DevCtl* C, bool ok) {
  if (ok) return 0;
  if (C->nbt >= C->max_bt) {
    C->stalled = 1;
    return 0;
  }
  C->s = __dmul_rn(C->s, C->beta);
  C->nbt++;
  return 1;
}

// Inner-loop test (R6: res(kkt1) ≤ tol stops) and, if continuing, the next direction's setup.
SSN_DEV int inner_next(DevCtl* C, const EvalOut* ev0, int64_t m, int nsm, int wsplits, int* info) {
  const int go = (C->numeric == 0) && (C->j < C->max_inner) && !(ev0->res1 <= C->tol_in);
  if (go) {
    C->geo = make_geo(ev0->r, m, nsm, wsplits, C->sc.kappa, C->kinv, C->cg_ratio, C->cg_threshold);
    C->geo.jit = C->retry ? C->jitter : 0.0;
    *info = 0;
  }
  return go;
}

// outer begin: σ-scalars, j = 0
__global__ void k_ctl_outer_begin(DevCtl* C) {
  C->sc = make_scal_dev(C->sigma, C->l1, C->l2);
  C->kinv = __ddiv_rn(1.0, C->sc.kappa);
  C->j = 0;
  C->seg_outer++;
}

// after EVAL at the outer start: first inner test
SSN_DEV void ctl_inner_begin(DevCtl* C, const EvalOut* ev0, int64_t m, int nsm, int wsplits, int* info,
                             cudaGraphConditionalHandle h_inner) {
  C->psi_evals++;
  C->tol_in = C->tol;
  if (C->inner_tol_mode) {  // res(kkt3), Eq. (20), of the point the outer iteration starts from
    const double res3 = __ddiv_rn(__ddiv_rn(__dsqrt_rn(ev0->s[1]), C->sigma),
                                  __dadd_rn(__dadd_rn(1.0, __dsqrt_rn(ev0->yy)), __dsqrt_rn(ev0->s[2])));
    C->tol_in = fmax(C->tol, __dmul_rn(0.1, res3));
  }
  cudaGraphSetConditional(h_inner, inner_next(C, ev0, m, nsm, wsplits, info));
}

// after the trial evaluation at s = 1: numeric checks, first Armijo test, K1 timing
SSN_DEV void ctl_armijo(DevCtl* C, const EvalOut* ev0, const EvalOut* ev1, cudaGraphConditionalHandle h_bt,
                        bool redo_pass = false) {
  if (C->tstamp[1] > C->tstamp[0]) {
    C->k1_ns += C->tstamp[1] - C->tstamp[0];
    C->k1_cnt++;
  }
  C->tstamp[0] = ~0ull;
  C->tstamp[1] = 0ull;
  if (redo_pass) {  // R40: the same trial, now streamed (bitwise the same ψ, with its ∇ψ): decide again
    C->redo = 0;
    cudaGraphSetConditional(h_bt, bt_next(C, armijo_ok(C, ev1->psi, ev0->psi, ev0->psimag)));
    return;
  }
  C->seg_inner++;
  C->psi_evals++;
  C->aty_passes++;
  C->branch_steps[C->geo.branch]++;
  C->nbt = 0;
  C->s = 1.0;
  const bool fac = C->geo.branch == 1 || C->geo.branch == 2;
  const bool failed = fac && (ev1->info != 0 || C->inject > 0);
  if (fac && C->inject > 0) C->inject--;
  if (failed && !C->retry && C->jitter > 0.0) {
    C->retry = 1;  // redo this step from the same y with the jittered factor (R36)
    C->skip = 1;
    C->need_grad = 0;
    C->jitter_retries++;
    cudaGraphSetConditional(h_bt, 0);
    return;
  }
  if (failed) {
    C->numeric = 1;
    C->numeric_kind = 1;
    C->numeric_r = C->geo.r;
  } else if (!isfinite(ev1->psi) || !isfinite(ev1->gd)) {
    C->numeric = 1;
    C->numeric_kind = 2;
  }
  if (C->numeric) {
    cudaGraphSetConditional(h_bt, 0);
    return;
  }
  C->gd = ev1->gd;
  const bool ok = armijo_ok(C, ev1->psi, ev0->psi, ev0->psimag);
  if (ok && C->gmiss) {  // R40: s = 1 accepted on a ψ-only trial: the redo nodes stream it (no decision yet)
    C->redo = 1;
    cudaGraphSetConditional(h_bt, 0);
    return;
  }
  cudaGraphSetConditional(h_bt, bt_next(C, ok));
}

// after a backtrack evaluation (no gradient) at the current s
SSN_DEV void ctl_bt(DevCtl* C, const EvalOut* ev0, const EvalOut* evb, cudaGraphConditionalHandle h_bt) {
  C->seg_bt++;
  C->psi_evals++;
  cudaGraphSetConditional(h_bt, bt_next(C, armijo_ok(C, evb->psi, ev0->psi, ev0->psimag)));
}

// Accept y ← y + s d (Algorithm 1 step (3)): trial → current.  nbt = 0: the trial's J, P_J, w,
// gradient and EvalOut are those of the accepted point; nbt > 0: J, P_J from the last K1e,
// w from the materialised w + s (w1 − w); the gradient is recomputed (need_grad).
__global__ void __launch_bounds__(256) k_accept(DevCtl* C, int64_t m, int64_t n, double* __restrict__ y0,
                                                const double* __restrict__ y1, double* __restrict__ g0,
                                                const double* __restrict__ g1, int32_t* __restrict__ J0,
                                                const int32_t* __restrict__ J1, double* __restrict__ P0,
                                                const double* __restrict__ P1, int64_t* r_dev,
                                                double* __restrict__ w0, const double* __restrict__ w1,
                                                const double* __restrict__ w2, EvalOut* ev) {
  if (C->numeric || C->skip) return;
  const int nb = C->nbt;
  const int64_t r1 = r_dev[1];
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
  const double* ws = nb == 0 ? w1 : w2;
  for (int64_t i = tid; i < n; i += nth) w0[i] = ws[i];
  for (int64_t i = tid; i < r1; i += nth) {
    J0[i] = J1[i];
    P0[i] = P1[i];
  }
  for (int64_t i = tid; i < m; i += nth) {
    y0[i] = y1[i];
    if (nb == 0) g0[i] = g1[i];
  }
  if (tid == 0) {
    r_dev[0] = r1;
    if (nb == 0) ev[0] = ev[1];
    C->backtracks += nb;
    C->newton_iters++;
    C->retry = 0;
    C->need_grad = nb > 0;
    if (nb > 0) C->seg_grad++;
  }
}

// end of a Newton step: next inner test
SSN_DEV void ctl_inner_end(DevCtl* C, const EvalOut* ev0, int64_t m, int nsm, int wsplits, int* info,
                           cudaGraphConditionalHandle h_inner) {
  if (C->skip) C->skip = 0;  // a retried step does not advance j (host: --j)
  else if (C->numeric == 0) C->j++;
  cudaGraphSetConditional(h_inner, inner_next(C, ev0, m, nsm, wsplits, info));
}

// x ← P (Eq. (10) via Moreau): after k_zero_at cleared the old support, scatter the new
// one and keep it as (Jx, Px, rx).
__global__ void __launch_bounds__(256) k_xupdate(const DevCtl* C, const int32_t* __restrict__ J0,
                                                 const double* __restrict__ P0, int64_t* r_dev,
                                                 double* __restrict__ x, int32_t* __restrict__ Jx,
                                                 double* __restrict__ Px) {
  if (C->numeric) return;
  const int64_t r = r_dev[0];
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = tid; i < r; i += nth) {
    const int32_t j = J0[i];
    const double v = P0[i];
    x[j] = v;
    Jx[i] = j;
    Px[i] = v;
  }
  if (tid == 0) r_dev[2] = r;
}

// outer end: res(kkt3) Eq. (20), stop test (R7), σ ← min(5σ, σmax) (R9)
__global__ void k_ctl_outer_end(DevCtl* C, const EvalOut* ev0, cudaGraphConditionalHandle h_outer) {
  if (C->numeric) {
    C->outer_iters = C->k;
    C->sigma_final = C->sigma;
    cudaGraphSetConditional(h_outer, 0);
    return;
  }
  const double sig = C->sigma;
  const double res3 = __ddiv_rn(__ddiv_rn(__dsqrt_rn(ev0->s[1]), sig),
                                __dadd_rn(__dadd_rn(1.0, __dsqrt_rn(ev0->yy)), __dsqrt_rn(ev0->s[2])));
  C->res3 = res3;
  C->res1 = ev0->res1;
  C->k++;
  if (res3 <= C->tol && ev0->res1 <= C->tol) {
    C->converged = 1;
    C->outer_iters = C->k;
    C->sigma_final = sig;
    cudaGraphSetConditional(h_outer, 0);
    return;
  }
  C->sigma = fmin(__dmul_rn(C->sigma_factor, sig), C->sigma_max);
  C->sigma_final = C->sigma;
  const int go = C->k < C->max_outer;
  if (!go) C->outer_iters = C->k;
  cudaGraphSetConditional(h_outer, go);
}

// ---- ψ evaluation fused with the control decision that consumes it (one graph node instead of
// two; each dependent node costs ~1-1.5 µs).  The finishing thread of the evaluation (EvalOut
// written) runs the decision; with KIND = kHookInnerEnd and the gradient recompute predicated
// off, thread 0 runs the decision alone.
struct CtlHook {
  DevCtl* C;
  const EvalOut* ev0;  // current point's record
  const EvalOut* ev1;  // this evaluation's record (Armijo trial / backtrack)
  int64_t m;
  int nsm, wsplits;
  int* info;
  cudaGraphConditionalHandle h;
};
enum { kHookInnerBegin = 1, kHookArmijo = 2, kHookBacktrack = 3, kHookInnerEnd = 4, kHookArmijoRedo = 5 };

template <int KIND>
__global__ void __cluster_dims__(kEvalCS, 1, 1) __launch_bounds__(K5_THREADS)
    k_eval_ctl(int64_t m, const double* __restrict__ y, const double* __restrict__ bvec,
               const double* __restrict__ part_vec, const int* __restrict__ part_valid, int nparts,
               const double* __restrict__ part_scal, int nscal, Scal sc, double nb, int with_grad,
               double* __restrict__ g_out, const int64_t* r_in, EvalOut* out, double* blk, unsigned* ticket,
               const double* gd_src, const int* info_src, EvalOut* host_out, unsigned long long seq, const Scal* scp,
               const int* pred, const double* nbp, CtlHook hk) {
  if (KIND == kHookInnerEnd && pred && *pred == 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) ctl_inner_end(hk.C, hk.ev0, hk.m, hk.nsm, hk.wsplits, hk.info, hk.h);
    return;
  }
  if (!eval_body(m, y, bvec, part_vec, part_valid, nparts, part_scal, nscal, sc, nb, with_grad, g_out, r_in, out, blk,
                 ticket, gd_src, info_src, host_out, seq, scp, pred, nbp))
    return;
  if (KIND == kHookInnerBegin) ctl_inner_begin(hk.C, hk.ev0, hk.m, hk.nsm, hk.wsplits, hk.info, hk.h);
  if (KIND == kHookArmijo) ctl_armijo(hk.C, hk.ev0, hk.ev1, hk.h);
  if (KIND == kHookArmijoRedo) ctl_armijo(hk.C, hk.ev0, hk.ev1, hk.h, true);
  if (KIND == kHookBacktrack) ctl_bt(hk.C, hk.ev0, hk.ev1, hk.h);
  if (KIND == kHookInnerEnd) ctl_inner_end(hk.C, hk.ev0, hk.m, hk.nsm, hk.wsplits, hk.info, hk.h);
}

// m ≤ 512: the same on one 16-CTA cluster (eval_body16)
template <int KIND>
__global__ void __cluster_dims__(kEval16, 1, 1) __launch_bounds__(K5_THREADS)
    k_eval_ctl16(int64_t m, const double* __restrict__ y, const double* __restrict__ bvec,
                 const double* __restrict__ part_vec, const int* __restrict__ part_valid, int nparts,
                 const double* __restrict__ part_scal, int nscal, Scal sc, double nb, int with_grad,
                 double* __restrict__ g_out, const int64_t* r_in, EvalOut* out, double* blk, unsigned* ticket,
                 const double* gd_src, const int* info_src, EvalOut* host_out, unsigned long long seq,
                 const Scal* scp, const int* pred, const double* nbp, CtlHook hk) {
  if (KIND == kHookInnerEnd && pred && *pred == 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) ctl_inner_end(hk.C, hk.ev0, hk.m, hk.nsm, hk.wsplits, hk.info, hk.h);
    return;
  }
  if (!eval_body16(m, y, bvec, part_vec, part_valid, nparts, part_scal, nscal, sc, nb, with_grad, g_out, r_in, out,
                   gd_src, info_src, host_out, seq, scp, pred, nbp))
    return;
  if (KIND == kHookInnerBegin) ctl_inner_begin(hk.C, hk.ev0, hk.m, hk.nsm, hk.wsplits, hk.info, hk.h);
  if (KIND == kHookArmijo) ctl_armijo(hk.C, hk.ev0, hk.ev1, hk.h);
  if (KIND == kHookArmijoRedo) ctl_armijo(hk.C, hk.ev0, hk.ev1, hk.h, true);
  if (KIND == kHookBacktrack) ctl_bt(hk.C, hk.ev0, hk.ev1, hk.h);
  if (KIND == kHookInnerEnd) ctl_inner_end(hk.C, hk.ev0, hk.m, hk.nsm, hk.wsplits, hk.info, hk.h);
}

}  // namespace ssn
