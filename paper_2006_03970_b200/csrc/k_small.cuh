// K7  k_small_solve: the whole of Algorithm 1 for small problems
// (m ≤ 64, n ≤ kSmallMaxN) in ONE thread block of 512 threads.
//
// For such problems every step of the hot path is latency-bound: a K1 pass over A is 0.4 MB at
// cfg1, the Newton systems are ≤ 64 × 64, and the graph path pays ~10 dependent kernels (each a
// few µs of launch, L2 round trips and grid-wide reductions) per Newton step.  Here the iterates
// (x, w, J, P_J, y, g, d) live in shared memory, A streams from L2 (it is L2-resident after the
// first pass), every reduction is a fixed-order block reduction, and the control decisions of
// Algorithm 1 are taken by every thread from the same shared values (no host round trip, no grid
// barrier).  The arithmetic follows the other paths operation by operation where the oracle fixes
// it (prox, Armijo with the roundoff guard R29, σ update, res1/res3, the SMW and m × m systems of
// Eq. (18)/(19), the factor retry R36); reduction orders differ, so results agree with the graph
// and host modes up to rounding (tests compare against the oracle, like those paths).
//
// Work per evaluation: w_i = a_iᵀy by a warp per column (lane ℓ holds rows ℓ and ℓ + 32, xor-butterfly
// sum), the epilogue of K1 on lane 0, a block scan for the ordered compaction of J, and
// ∇ψ = y + b − A_J P_J with warps over J.  Newton systems: the Gram from A_J staged in shared
// memory, a right-looking Cholesky (one warp scales the pivot column, the block updates the
// trailing part) with the right-hand side as row N, and a one-warp backward substitution.
#pragma once
#include "k_ctl.cuh"

namespace ssn {

constexpr int kSmallMaxM = 64;
constexpr int kSmallMaxN = 1024;
constexpr int kSmallChunk = 64;  // columns per TMA chunk of a pass (≤ 32 KB at m = 64)
constexpr int kSmallThreads = 512;
constexpr int kSmallNW = kSmallThreads / 32;       // warps
constexpr int kSmallCPT = kSmallMaxN / kSmallThreads;  // columns per thread in the epilogue
constexpr int kSmallLd = kSmallMaxM + 2;  // Newton matrix leading dimension (N + 1 ≤ 65 rows)

#ifdef SMALL_PROF  // phase cycle totals (thread 0): pass, epilogue, gradient, gram, factor, backward+d, control
__device__ unsigned long long g_small_prof[8];
#define SPROF_T0() long long sp_t0_ = clock64()
#define SPROF_ADD(k) do { if (tid == 0) { const long long t_ = clock64(); g_small_prof[k] += t_ - sp_t0_; sp_t0_ = t_; } } while (0)
#else
#define SPROF_T0() do {} while (0)
#define SPROF_ADD(k) do {} while (0)
#endif

struct SmallParams {
  const double* A;  // m × n column-major (lda = m)
  const double* b;
  int m, n;
  double* x;        // in: x after init_point (dense); out: final x
  double* y0;       // initial y (init_point); on exit the final y (the next path point starts there, R39)
  double* w0;       // initial w = Aᵀy0 (0 when cold); on exit the final w
  int32_t* Jx;      // out: support of x (ascending) and its values, count
  double* Px;
  int64_t* rx;
  DevCtl* C;        // settings in, statistics out
  EvalOut* ev;      // out: evaluation at the final point (dual objective)
  // k_small_cl only (the one-CTA kernel leaves them to the multi-kernel helpers):
  int cold;         // 1: x0 = 0 (y0 = 0, w0 = 0, x = 0 are not read; *rx0 ← 0)
  int64_t* rx0;     // |supp x0| for the statistics
  double* obj;      // out: [½‖Ax − b‖², Σ|x|, Σx², nnz] of the final x (nullable)
  double* resid;    // out: A x − b (m), for the certify pass (nullable)
  // k_small_cl launch-overhead trims (nullable / 0 = off): settings by value instead of an H2D copy of
  // the control block, the carried σ0 read from the device, results written straight into the
  // caller's mapped pinned host mirrors and the caller's device x buffer (no copies after the launch)
  int use_cin;
  DevCtl cin;
  const double* sigma_in;
  DevCtl* cout_host;
  EvalOut* ev_host;
  double* rx0_host;  // |supp x0| as int64 bits (scratch slot 20)
  double* xout;
};

// shared-memory layout (doubles unless noted)
constexpr size_t kSmallSmem =
    (size_t)8 * (3 * kSmallMaxN      // w[3]
                 + kSmallMaxN        // x
                 + 2 * kSmallMaxN    // PJ[2]
                 + (kSmallMaxM + 1) * kSmallLd  // Newton matrix (column-major, ld = kSmallLd; L in its upper part)
                 + 2 * kSmallMaxM    // diag(L) and its inverse
                 + kSmallMaxM * kSmallMaxM  // A_J staging (column a at a·m)
                 + kSmallNW * kSmallMaxM  // per-warp m-vector partials
                 + 8 * kSmallMaxM    // y[2], g[2], d, yt, v, spare
                 + 64 + kSmallNW * 4  // scalars, per-warp scalar partials
                 + 2 * kSmallChunk * kSmallMaxM  // A chunk ring (2 stages)
                 + 2)                // mbarriers
    + (size_t)4 * (2 * kSmallMaxN + 64);  // J[2] (int32), scan scratch

__global__ void __launch_bounds__(kSmallThreads, 1) k_small_solve(const SmallParams p) {
  extern __shared__ __align__(16) double sm[];
  const int m = p.m, n = p.n;
  double* w = sm;                                   // w[q] = sm + q·kSmallMaxN
  double* xs = w + 3 * kSmallMaxN;
  double* PJs = xs + kSmallMaxN;                    // PJ[c] = PJs + c·kSmallMaxN
  double* Mx = PJs + 2 * kSmallMaxN;                // Mx[i + c·kSmallLd]
  double* Ld = Mx + (kSmallMaxM + 1) * kSmallLd;    // L_jj, then 1/L_jj at Ld + 64
  double* AJ = Ld + 2 * kSmallMaxM;                 // AJ[a·m + k] = A[k, J_a]
  double* red = AJ + kSmallMaxM * kSmallMaxM;       // red[warp·64 + k]
  double* ys = red + kSmallNW * kSmallMaxM;         // y[c] = ys + c·64
  double* gs = ys + 2 * kSmallMaxM;                 // g[c] = gs + c·64
  double* ds = gs + 2 * kSmallMaxM;                 // d
  double* vs = ds + kSmallMaxM;                     // v (solve), b
  double* bs = vs + kSmallMaxM;
  double* yt = bs + kSmallMaxM;                     // trial / backtrack point
  double* sc_ = yt + kSmallMaxM;                    // scalars (broadcast)
  double* wred = sc_ + 64;                          // per-warp scalar partials [32][4]
  double* ring = wred + kSmallNW * 4;               // stage q at ring + q·kSmallChunk·64
  uint64_t* fullb = (uint64_t*)(ring + 2 * kSmallChunk * kSmallMaxM);
  int32_t* Js = (int32_t*)(fullb + 2);              // J[c] = Js + c·kSmallMaxN
  int* iscr = Js + 2 * kSmallMaxN;                  // scan scratch (warp totals)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr unsigned FULL = 0xffffffffu;

  // ---- settings and state ----
  __shared__ DevCtl C;
  if (tid == 0) {
    C = *p.C;
    mbar_init(fullb, 1);
    mbar_init(fullb + 1, 1);
    fence_mbar_init();
  }
  uint32_t nfill = 0;  // chunks issued so far (all threads track it: parity of each stage)
  for (int i = tid; i < n; i += kSmallThreads) {
    xs[i] = p.x[i];
    w[i] = p.w0[i];
  }
  if (tid < m) {
    ys[tid] = p.y0[tid];
    bs[tid] = p.b[tid];
  }
  __syncthreads();
  const double l1 = C.l1, l2 = C.l2, tol = C.tol, nb = C.nb;

  // Σ over the block in a fixed order: per-warp partials (lane 0 of warp q holds v) → thread 0.
  // Returns the sum to every thread.
  auto block_sum4 = [&](double (&v)[4]) {
    if (lane == 0)
      for (int j = 0; j < 4; ++j) wred[warp * 4 + j] = v[j];
    __syncthreads();
    if (tid == 0) {
      double s[4] = {0, 0, 0, 0};
      for (int q = 0; q < kSmallNW; ++q)
        for (int j = 0; j < 4; ++j) s[j] = __dadd_rn(s[j], wred[q * 4 + j]);
      for (int j = 0; j < 4; ++j) sc_[j] = s[j];
    }
    __syncthreads();
    for (int j = 0; j < 4; ++j) v[j] = sc_[j];
    __syncthreads();
  };

  // w_dst = Aᵀ y over all n columns: chunks of 64 consecutive columns (contiguous in column-major A)
  // stream L2 → shared memory by 1D bulk copies (TMA) through a 2-stage ring; per chunk thread t
  // takes column t/8 and rows ≡ t (mod 8), three shuffles finish each column (fixed order)
  auto pass = [&](const double* yv, double* wdst) {
    SPROF_T0();
    const int nch = (n + kSmallChunk - 1) / kSmallChunk;
    const int kk = tid & 7, cc = tid >> 3;
    // Two chunks in flight; a chunk's stage is refilled after every thread has used it.
    uint32_t base = nfill;
    if (tid == 0) {
      for (int ch = 0; ch < min(2, nch); ++ch) {
        const int c0 = ch * kSmallChunk, nc = min(kSmallChunk, n - c0);
        const uint32_t bytes = (uint32_t)nc * m * 8;
        const uint32_t st = (base + ch) & 1;
        double* dst = ring + st * kSmallChunk * kSmallMaxM;
        if (bytes % 16 == 0) {
          mbar_arrive_expect_tx(fullb + st, bytes);
          bulk_g2s(dst, p.A + (int64_t)c0 * m, bytes, fullb + st);
        } else {
          dst[nc * m - 1] = p.A[(int64_t)c0 * m + nc * m - 1];
          mbar_arrive_expect_tx(fullb + st, bytes - 8);
          if (bytes > 8) bulk_g2s(dst, p.A + (int64_t)c0 * m, bytes - 8, fullb + st);
        }
      }
    }
    for (int ch = 0; ch < nch; ++ch) {
      const uint32_t st = (base + ch) & 1, par = ((base + ch) >> 1) & 1;
      mbar_wait(fullb + st, par);
      const double* S = ring + st * kSmallChunk * kSmallMaxM;
      const int c0 = ch * kSmallChunk, nc = min(kSmallChunk, n - c0);
      double s0 = 0.0, s1 = 0.0;
      if (cc < nc) {
#pragma unroll
        for (int q = 0; q < 8; q += 2) {
          const int k0 = kk + 8 * q, k1 = k0 + 8;
          if (k0 < m) s0 = __fma_rn(S[cc * m + k0], yv[k0], s0);
          if (k1 < m) s1 = __fma_rn(S[cc * m + k1], yv[k1], s1);
        }
      }
      double v = __dadd_rn(s0, s1);
      v = __dadd_rn(v, __shfl_xor_sync(FULL, v, 4));
      v = __dadd_rn(v, __shfl_xor_sync(FULL, v, 2));
      v = __dadd_rn(v, __shfl_xor_sync(FULL, v, 1));
      if (kk == 0 && cc < nc) wdst[c0 + cc] = v;
      __syncthreads();  // every thread is done with stage st
      if (tid == 0 && ch + 2 < nch) {
        const int c2 = (ch + 2) * kSmallChunk, nc2 = min(kSmallChunk, n - c2);
        const uint32_t bytes = (uint32_t)nc2 * m * 8;
        double* dst = ring + st * kSmallChunk * kSmallMaxM;
        if (bytes % 16 == 0) {
          mbar_arrive_expect_tx(fullb + st, bytes);
          bulk_g2s(dst, p.A + (int64_t)c2 * m, bytes, fullb + st);
        } else {
          dst[nc2 * m - 1] = p.A[(int64_t)c2 * m + nc2 * m - 1];
          mbar_arrive_expect_tx(fullb + st, bytes - 8);
          if (bytes > 8) bulk_g2s(dst, p.A + (int64_t)c2 * m, bytes - 8, fullb + st);
        }
      }
    }
    nfill = base + nch;
    __syncthreads();
    SPROF_ADD(0);
  };

  // Epilogue of K1/K1e at σ-scalars s: w_eff = w0 (+ step (w1 − w0)) [stored to wout], t = x − σ w,
  // P = prox, ordered compaction → (J, P_J, r), partial sums s[0..3] (Σ P², Σ(x−P)², Σz², Σ(|w|−λ1)₊²).
  auto epilogue = [&](const Scal& sc, const double* w0p, const double* w1p, double step, double* wout, int jc,
                      double (&sums)[4]) -> int {
    // each thread owns kSmallCPT consecutive columns (n ≤ kSmallMaxN): flags, then a block scan
    SPROF_T0();
    const int i0 = kSmallCPT * tid;
    double wv[kSmallCPT], Pv[kSmallCPT];
    int act[kSmallCPT];
    double s[4] = {0, 0, 0, 0};
#pragma unroll
    for (int u = 0; u < kSmallCPT; ++u) {
      const int i = i0 + u;
      act[u] = 0;
      Pv[u] = 0.0;
      wv[u] = 0.0;
      if (i < n) {
        double ww = w0p[i];
        if (w1p) ww = __dadd_rn(ww, __dmul_rn(step, __dsub_rn(w1p[i], ww)));
        wv[u] = ww;
        const double xi = xs[i];
        const double tt = __dsub_rn(xi, __dmul_rn(sc.sigma, ww));
        act[u] = fabs(tt) > sc.thr;
        const double P = prox_en(tt, sc.thr, sc.den);
        Pv[u] = P;
        const double dx = __dsub_rn(xi, P);
        const double z = __dsub_rn(__ddiv_rn(dx, sc.sigma), ww);
        const double e = __dsub_rn(fabs(ww), sc.l1);
        s[0] = __dadd_rn(s[0], __dmul_rn(P, P));
        s[1] = __dadd_rn(s[1], __dmul_rn(dx, dx));
        s[2] = __dadd_rn(s[2], __dmul_rn(z, z));
        if (e > 0.0) s[3] = __dadd_rn(s[3], __dmul_rn(e, e));
      }
    }
    if (wout)
#pragma unroll
      for (int u = 0; u < kSmallCPT; ++u)
        if (i0 + u < n) wout[i0 + u] = wv[u];
    // warp sums of the scalar partials (butterfly, then fixed warp order in block_sum4)
#pragma unroll
    for (int j = 0; j < 4; ++j) s[j] = warp_allsum(s[j]);
    // scan of the active counts
    int cnt = 0;
#pragma unroll
    for (int u = 0; u < kSmallCPT; ++u) cnt += act[u];
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) iscr[warp] = incl;
    block_sum4(s);  // contains __syncthreads: iscr visible afterwards
    int off = 0, tot = 0;
    for (int q = 0; q < kSmallNW; ++q) {
      const int v = iscr[q];
      off += q < warp ? v : 0;
      tot += v;
    }
    int pos = off + incl - cnt;
    int32_t* Jd = Js + jc * kSmallMaxN;
    double* Pd = PJs + jc * kSmallMaxN;
#pragma unroll
    for (int u = 0; u < kSmallCPT; ++u)
      if (act[u]) {
        Jd[pos] = i0 + u;
        Pd[pos] = Pv[u];
        ++pos;
      }
    for (int j = 0; j < 4; ++j) sums[j] = s[j];
    __syncthreads();
    SPROF_ADD(1);
    return tot;
  };

  // g = y + b − A_J P_J and (yy, by, gg); returns via out[0..2]
  auto gradient = [&](const double* yv, int jc, int r, double* gdst, double (&out)[3], bool with_grad) {
    const int32_t* Jd = Js + jc * kSmallMaxN;
    const double* Pd = PJs + jc * kSmallMaxN;
    SPROF_T0();
    if (with_grad) {  // thread (k, part): Σ over a ≡ part (mod kParts) of P_a A[k, J_a], coalesced over k
      constexpr int kParts = kSmallThreads / kSmallMaxM;
      const int k = tid % kSmallMaxM, part = tid / kSmallMaxM;
      double a0 = 0.0, a1 = 0.0;
      if (k < m) {
        int a = part;
#pragma unroll 2
        for (; a + kParts < r; a += 2 * kParts) {
          a0 = __fma_rn(Pd[a], __ldg(p.A + (int64_t)Jd[a] * m + k), a0);
          a1 = __fma_rn(Pd[a + kParts], __ldg(p.A + (int64_t)Jd[a + kParts] * m + k), a1);
        }
        if (a < r) a0 = __fma_rn(Pd[a], __ldg(p.A + (int64_t)Jd[a] * m + k), a0);
      }
      red[part * kSmallMaxM + k] = __dadd_rn(a0, a1);
      __syncthreads();
    }
    if (warp == 0) {
      double yy = 0.0, by = 0.0, gg = 0.0;
      for (int h = 0; h < 2; ++h) {
        const int k = lane + 32 * h;
        if (k < m) {
          const double yk = yv[k], bk = bs[k];
          yy = __dadd_rn(yy, __dmul_rn(yk, yk));
          by = __dadd_rn(by, __dmul_rn(bk, yk));
          if (with_grad) {
            double gp = 0.0;
            for (int q = 0; q < kSmallThreads / kSmallMaxM; ++q) gp = __dadd_rn(gp, red[q * kSmallMaxM + k]);
            const double g = __dsub_rn(__dadd_rn(yk, bk), gp);
            gdst[k] = g;
            gg = __dadd_rn(gg, __dmul_rn(g, g));
          }
        }
      }
      yy = warp_allsum(yy);
      by = warp_allsum(by);
      gg = warp_allsum(gg);
      if (lane == 0) {
        sc_[8] = yy;
        sc_[9] = by;
        sc_[10] = gg;
      }
    }
    __syncthreads();
    out[0] = sc_[8];
    out[1] = sc_[9];
    out[2] = sc_[10];
    __syncthreads();
    SPROF_ADD(2);
  };

  // EvalOut at (y, sums, yy/by/gg)
  auto make_ev = [&](const Scal& sc, const double (&s)[4], const double (&q)[3], int r, bool with_grad) {
    EvalOut o;
    o.yy = q[0];
    o.by = q[1];
    o.gg = q[2];
    for (int j = 0; j < 4; ++j) o.s[j] = s[j];
    const double tprox = __dmul_rn(sc.cpsi, s[0]);
    o.psi = __dadd_rn(__dadd_rn(__dmul_rn(0.5, q[0]), q[1]), tprox);
    o.psimag = fabs(0.5 * q[0]) + fabs(q[1]) + fabs(tprox);
    o.res1 = with_grad ? sqrt(q[2]) / (1.0 + nb) : -1.0;
    o.gd = 0.0;
    o.r = r;
    o.info = 0;
    o.seq = 0;
    o.pad = 0;
    return o;
  };

  // Newton direction at (y = ys[cur], g = gs[cur], J[cur]): d (ds), gᵀd, branch; false on a bad pivot
  auto direction = [&](int cur, int r, double kappa, double jit, double& gd, int& br) -> bool {
    const double* g = gs + cur * kSmallMaxM;
    const int32_t* Jd = Js + cur * kSmallMaxN;
    SPROF_T0();
    if (r == 0) {
      br = 0;
      if (tid < m) ds[tid] = -g[tid];
    } else {
      const bool smw = r < m;
      br = smw ? 1 : 2;
      const int N = smw ? r : m;
      // ---- Gram (lower triangle) and right-hand side row N ----
      if (smw) {  // Eq. (19): κ⁻¹ I_r + A_Jᵀ A_J, rhs u = A_Jᵀ g
        for (int a = warp; a < r; a += kSmallNW) {
          const double* col = p.A + (int64_t)Jd[a] * m;
          if (lane < m) AJ[a * m + lane] = __ldg(col + lane);
          if (lane + 32 < m) AJ[a * m + lane + 32] = __ldg(col + lane + 32);
        }
        __syncthreads();
        const int npair = N * (N + 1) / 2;
        for (int e = tid; e < npair + N; e += kSmallThreads) {
          int i, c;
          const double* bc;
          if (e < npair) {  // (i, c), i ≥ c: row-major enumeration of the lower triangle
            i = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
            while ((i + 1) * (i + 2) / 2 <= e) ++i;
            while (i * (i + 1) / 2 > e) --i;
            c = e - i * (i + 1) / 2;
            bc = AJ + c * m;
          } else {
            i = N;
            c = e - npair;
            bc = g;
          }
          const double* ai = AJ + (i < N ? i : c) * m;
          double s0 = 0.0, s1 = 0.0;
          int k = 0;
          for (; k + 1 < m; k += 2) {
            s0 = __fma_rn(ai[k], bc[k], s0);
            s1 = __fma_rn(ai[k + 1], bc[k + 1], s1);
          }
          if (k < m) s0 = __fma_rn(ai[k], bc[k], s0);
          const double s = __dadd_rn(s0, s1);
          double v = s;
          if (i < N && i == c) {
            v = __dadd_rn(s, 1.0 / kappa);
            if (jit != 0.0) v = __fma_rn(v, jit, v);
          }
          Mx[i + c * kSmallLd] = v;
        }
      } else {  // Eq. (18): I_m + κ A_J A_Jᵀ, rhs g
        const int npair = m * (m + 1) / 2;
        constexpr int kPP = (kSmallMaxM * (kSmallMaxM + 1) / 2 + kSmallThreads - 1) / kSmallThreads;
        double acc[kPP];  // ≤ 2080 pairs
#pragma unroll
        for (int q = 0; q < kPP; ++q) acc[q] = 0.0;
        for (int a0 = 0; a0 < r; a0 += kSmallMaxM) {
          const int na = min(kSmallMaxM, r - a0);
          __syncthreads();
          for (int a = warp; a < na; a += kSmallNW) {
            const double* col = p.A + (int64_t)Jd[a0 + a] * m;
            if (lane < m) AJ[a * m + lane] = __ldg(col + lane);
            if (lane + 32 < m) AJ[a * m + lane + 32] = __ldg(col + lane + 32);
          }
          __syncthreads();
#pragma unroll
          for (int q = 0; q < kPP; ++q) {
            const int e = tid + q * kSmallThreads;
            if (e >= npair) break;
            int i = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
            while ((i + 1) * (i + 2) / 2 <= e) ++i;
            while (i * (i + 1) / 2 > e) --i;
            const int c = e - i * (i + 1) / 2;
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
            int a = 0;
            for (; a + 3 < na; a += 4) {
              s0 = __fma_rn(AJ[a * m + i], AJ[a * m + c], s0);
              s1 = __fma_rn(AJ[(a + 1) * m + i], AJ[(a + 1) * m + c], s1);
              s2 = __fma_rn(AJ[(a + 2) * m + i], AJ[(a + 2) * m + c], s2);
              s3 = __fma_rn(AJ[(a + 3) * m + i], AJ[(a + 3) * m + c], s3);
            }
            for (; a < na; ++a) s0 = __fma_rn(AJ[a * m + i], AJ[a * m + c], s0);
            acc[q] = __dadd_rn(acc[q], __dadd_rn(__dadd_rn(s0, s1), __dadd_rn(s2, s3)));
          }
        }
#pragma unroll
        for (int q = 0; q < kPP; ++q) {
          const int e = tid + q * kSmallThreads;
          if (e >= npair) break;
          int i = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
          while ((i + 1) * (i + 2) / 2 <= e) ++i;
          while (i * (i + 1) / 2 > e) --i;
          const int c = e - i * (i + 1) / 2;
          double v = __dadd_rn(__dmul_rn(kappa, acc[q]), i == c ? 1.0 : 0.0);
          if (i == c && jit != 0.0) v = __fma_rn(v, jit, v);
          Mx[i + c * kSmallLd] = v;
        }
        if (tid < m) Mx[m + tid * kSmallLd] = g[tid];
      }
      __syncthreads();
      SPROF_ADD(3);
      // ---- Cholesky with the rhs as row N (forward substitution for free), TWO pivots per barrier:
      // every thread recomputes the 2 × 2 diagonal block's factor (L_jj, L_{j+1,j}, L_{j+1,j+1}) from
      // the shared values and applies the rank-2 update to its entries; L[i][j] (i > j, incl. the rhs
      // row N) goes to the unused upper triangle Mx[j + i·ld], the Schur complement stays in the
      // lower one.  Thread t: row i = j + 2 + (t mod 64), columns c ≡ j + 2 + t/64 (mod 8), c ≤ i.
      {
        constexpr int kFW = kSmallThreads / 64;
        const int ti = tid & 63, tc = tid >> 6;
        int badl = 0;
        for (int j = 0; j < N; j += 2) {
          const bool two = j + 1 < N;
          const double a = Mx[j + j * kSmallLd];
          const bool ok0 = a > 0.0;
          const double d0 = ok0 ? a : 1.0;
          const double inv0 = rsqrt_pos(d0);
          double l10 = 0.0, d1 = 1.0, inv1 = 1.0;
          bool ok1 = true;
          if (two) {
            l10 = __dmul_rn(Mx[j + 1 + j * kSmallLd], inv0);
            const double c1 = __fma_rn(-l10, l10, Mx[j + 1 + (j + 1) * kSmallLd]);
            ok1 = c1 > 0.0;
            d1 = ok1 ? c1 : 1.0;
            inv1 = rsqrt_pos(d1);
          }
          badl |= !ok0 || !ok1;
          const int jn = two ? j + 2 : j + 1;  // first row / column after the block
          if (!two && tid <= N - jn) {  // single last pivot: column j of the rows below (incl. rhs)
            const int i = jn + tid;
            Mx[j + i * kSmallLd] = __dmul_rn(Mx[i + j * kSmallLd], inv0);
          }
          const int i = jn + ti;
          if (two && i <= N) {
            const double li0 = __dmul_rn(Mx[i + j * kSmallLd], inv0);
            const double li1 = __dmul_rn(__fma_rn(-li0, l10, Mx[i + (j + 1) * kSmallLd]), inv1);
            if (tc == 0) {
              Mx[j + i * kSmallLd] = li0;
              Mx[j + 1 + i * kSmallLd] = li1;
            }
            constexpr int kQ = 64 / kFW;
            double m0[kQ], m1[kQ], mc[kQ];
#pragma unroll
            for (int q = 0; q < kQ; ++q) {  // loads first, then the rank-2 updates
              const int c = jn + tc + kFW * q;
              const bool ok = c <= i && c < N;
              m0[q] = ok ? Mx[c + j * kSmallLd] : 0.0;
              m1[q] = ok ? Mx[c + (j + 1) * kSmallLd] : 0.0;
              mc[q] = ok ? Mx[i + c * kSmallLd] : 0.0;
            }
#pragma unroll
            for (int q = 0; q < kQ; ++q) {
              const int c = jn + tc + kFW * q;
              if (c <= i && c < N) {
                const double lc0 = __dmul_rn(m0[q], inv0);
                const double lc1 = __dmul_rn(__fma_rn(-lc0, l10, m1[q]), inv1);
                Mx[i + c * kSmallLd] = __fma_rn(-li1, lc1, __fma_rn(-li0, lc0, mc[q]));
              }
            }
          }
          if (tid == 0) {
            Ld[j] = __dmul_rn(d0, inv0);
            Ld[kSmallMaxM + j] = inv0;
            if (two) {
              Mx[j + (j + 1) * kSmallLd] = l10;
              Ld[j + 1] = __dmul_rn(d1, inv1);
              Ld[kSmallMaxM + j + 1] = inv1;
            }
          }
          __syncthreads();
        }
        if (tid == 0 && badl) sc_[16] = 1.0;
        __syncthreads();
      }
      SPROF_ADD(4);
      const int bad = sc_[16] != 0.0;
      // ---- backward substitution v = L⁻ᵀ z (z = row N), one warp; rows lane and lane + 32 ----
      if (warp == 0) {
        double z0 = lane < N ? Mx[lane + N * kSmallLd] : 0.0, z1 = lane + 32 < N ? Mx[lane + 32 + N * kSmallLd] : 0.0;
        for (int i = N - 1; i >= 0; --i) {
          const double zi = __shfl_sync(FULL, i < 32 ? z0 : z1, i & 31);
          const double vi = __dmul_rn(zi, Ld[kSmallMaxM + i]);
          if (lane == (i & 31)) {
            if (i < 32) z0 = vi;
            else z1 = vi;
          }
          // z_k −= L[i][k] v_i for k < i (L[i][k] at Mx[k + i·ld])
          if (lane < i) z0 = __fma_rn(-Mx[lane + i * kSmallLd], vi, z0);
          if (lane + 32 < i) z1 = __fma_rn(-Mx[lane + 32 + i * kSmallLd], vi, z1);
        }
        if (lane < N) vs[lane] = z0;
        if (lane + 32 < N) vs[lane + 32] = z1;
      }
      __syncthreads();
      if (smw) {  // d = −g + A_J v
        if (tid < m) {
          double s = 0.0;
          for (int a = 0; a < r; ++a) s = __dadd_rn(s, __dmul_rn(AJ[a * m + tid], vs[a]));
          ds[tid] = __dadd_rn(-g[tid], s);
        }
      } else {  // d = −M⁻¹ g
        if (tid < m) ds[tid] = -vs[tid];
      }
      if (bad) {
        __syncthreads();
        if (tid == 0) sc_[16] = 0.0;
        __syncthreads();
        return false;
      }
    }
    __syncthreads();
    if (warp == 0) {
      double s = 0.0;
      for (int h = 0; h < 2; ++h) {
        const int k = lane + 32 * h;
        if (k < m) s = __dadd_rn(s, __dmul_rn(g[k], ds[k]));
      }
      s = warp_allsum(s);
      if (lane == 0) sc_[11] = s;
    }
    __syncthreads();
    gd = sc_[11];
    __syncthreads();
    SPROF_ADD(5);
    return true;
  };

  // ---- Algorithm 1 ----
  if (tid == 0) sc_[16] = 0.0;
  int cur = 0, wcur = 0;
  double sigma = C.sigma;
  int converged = 0, numeric = 0, numeric_kind = 0, stalled = 0;
  int newton = 0, psi_evals = 0, backtracks = 0, aty = 0, jretries = 0;
  int brs[4] = {0, 0, 0, 0};
  int inject = C.inject;
  double res1 = 0.0, res3 = 0.0;
  long long numeric_r = 0;
  EvalOut ev;
  int r_cur = 0;
  int k;
  for (k = 0; k < C.max_outer && !numeric; ++k) {
    const Scal sc = make_scal_dev(sigma, l1, l2);
    double s4[4], q3[3];
    r_cur = epilogue(sc, w + wcur * kSmallMaxN, nullptr, 0.0, nullptr, cur, s4);
    gradient(ys + cur * kSmallMaxM, cur, r_cur, gs + cur * kSmallMaxM, q3, true);
    ev = make_ev(sc, s4, q3, r_cur, true);
    psi_evals++;
    double tol_in = tol;
    if (C.inner_tol_mode) {
      const double res3_0 = (sqrt(ev.s[1]) / sigma) / (1.0 + sqrt(ev.yy) + sqrt(ev.s[2]));
      tol_in = fmax(tol, 0.1 * res3_0);
    }
    int retry = 0;
    for (int j = 0; j < C.max_inner; ++j) {
      if (ev.res1 <= tol_in) break;
      const int tr = 1 - cur;
      const int wtr = (wcur + 1) % 3, wbt = (wcur + 2) % 3;
      double gd = 0.0;
      int br = 0;
      bool fok = direction(cur, r_cur, sc.kappa, retry ? C.jitter : 0.0, gd, br);
      brs[br]++;
      // trial s = 1: y_t = y + d, full pass
      if (tid < m) ys[tr * kSmallMaxM + tid] = __dadd_rn(ys[cur * kSmallMaxM + tid], ds[tid]);
      __syncthreads();
      pass(ys + tr * kSmallMaxM, w + wtr * kSmallMaxN);
      aty++;
      double st4[4], qt3[3];
      const int r_t = epilogue(sc, w + wtr * kSmallMaxN, nullptr, 0.0, nullptr, tr, st4);
      gradient(ys + tr * kSmallMaxM, tr, r_t, gs + tr * kSmallMaxM, qt3, true);
      EvalOut evt = make_ev(sc, st4, qt3, r_t, true);
      psi_evals++;
      int info = fok ? 0 : 1;
      if ((br == 1 || br == 2) && inject > 0) {
        inject--;
        info = 1;
      }
      if ((br == 1 || br == 2) && info != 0 && !retry && C.jitter > 0.0) {
        retry = 1;
        jretries++;
        --j;
        continue;
      }
      if ((br == 1 || br == 2) && info != 0) {
        numeric = 1;
        numeric_kind = 1;
        numeric_r = r_cur;
        break;
      }
      if (!isfinite(evt.psi) || !isfinite(gd)) {
        numeric = 1;
        numeric_kind = 2;
        break;
      }
      double s = 1.0;
      int nbt = 0;
      auto armijo = [&](double psi_t) {
        const double lhs = __dsub_rn(psi_t, ev.psi);
        const double rhs = __dadd_rn(__dmul_rn(__dmul_rn(C.mu, s), gd), __dmul_rn(__dmul_rn(10.0, kEpsDev), ev.psimag));
        return lhs <= rhs;
      };
      bool ok = armijo(evt.psi);
      while (!ok) {
        if (nbt >= C.max_bt) {
          stalled = 1;  // R30: accept the last s
          break;
        }
        s = __dmul_rn(s, C.beta);
        nbt++;
        if (tid < m) ys[tr * kSmallMaxM + tid] = __fma_rn(s, ds[tid], ys[cur * kSmallMaxM + tid]);
        __syncthreads();
        double sb4[4], qb3[3];
        const int r_b = epilogue(sc, w + wcur * kSmallMaxN, w + wtr * kSmallMaxN, s, w + wbt * kSmallMaxN, tr, sb4);
        gradient(ys + tr * kSmallMaxM, tr, r_b, nullptr, qb3, false);
        evt = make_ev(sc, sb4, qb3, r_b, false);
        psi_evals++;
        ok = armijo(evt.psi);
      }
      backtracks += nbt;
      if (nbt == 0) {
        cur = tr;
        wcur = wtr;
        ev = evt;
        r_cur = r_t;
      } else {  // the accepted point needs ∇ψ for its re-thresholded J
        cur = tr;
        wcur = wbt;
        r_cur = (int)evt.r;
        double q2[3];
        gradient(ys + cur * kSmallMaxM, cur, r_cur, gs + cur * kSmallMaxM, q2, true);
        ev = make_ev(sc, evt.s, q2, r_cur, true);
      }
      newton++;
      retry = 0;
    }
    if (numeric) break;
    res3 = (sqrt(ev.s[1]) / sigma) / (1.0 + sqrt(ev.yy) + sqrt(ev.s[2]));
    res1 = ev.res1;
    // multiplier update Eq. (10): x ← P
    for (int i = tid; i < n; i += kSmallThreads) xs[i] = 0.0;
    __syncthreads();
    for (int a = tid; a < r_cur; a += kSmallThreads) {
      const int32_t i = Js[cur * kSmallMaxN + a];
      const double v = PJs[cur * kSmallMaxN + a];
      xs[i] = v;
      p.Jx[a] = i;  // support of x (objective, warm starts)
      p.Px[a] = v;
    }
    if (tid == 0) *p.rx = r_cur;
    __syncthreads();
    if (res3 <= tol && ev.res1 <= tol) {
      converged = 1;
      k++;
      break;
    }
    sigma = fmin(C.sigma_factor * sigma, C.sigma_max);
  }
  // ---- outputs ----  (x; and the final dual iterate y, w = Aᵀy, which the next point of a path starts
  // from under reading R39 — y0 / w0 were read at the start, so overwriting them is safe)
  for (int i = tid; i < n; i += kSmallThreads) {
    p.x[i] = xs[i];
    p.w0[i] = w[wcur * kSmallMaxN + i];
  }
  if (tid < m) p.y0[tid] = ys[cur * kSmallMaxM + tid];
  if (tid == 0) {
    DevCtl* o = p.C;
    o->outer_iters = k;
    o->newton_iters = newton;
    o->psi_evals = psi_evals;
    o->backtracks = backtracks;
    o->aty_passes = aty;
    for (int q = 0; q < 4; ++q) o->branch_steps[q] = brs[q];
    o->cg_iters = 0;
    o->jitter_retries = jretries;
    o->stalled = stalled;
    o->res1 = res1;
    o->res3 = res3;
    o->sigma_final = sigma;
    o->converged = converged;
    o->numeric = numeric;
    o->numeric_kind = numeric_kind;
    o->numeric_r = numeric_r;
    o->seg_outer = o->seg_inner = o->seg_bt = o->seg_grad = 0;
    o->k1_ns = 0;
    o->k1_cnt = 0;
    *p.ev = ev;
  }
}

}  // namespace ssn
