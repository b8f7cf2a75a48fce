// K7c  k_small_cl: the whole of Algorithm 1 for small problems
// (m ≤ 64, n ≤ 1024) on ONE 16-CTA thread-block cluster.
//
// The one-CTA kernel (k_small.cuh) streams A from L2 on a single SM every pass (~45 GB/s: ~9 µs
// per pass at cfg1) and factors the Newton matrix with one block barrier per two pivots.  Here A is
// RESIDENT in distributed shared memory: CTA q keeps its column block [q·n/16, (q+1)·n/16) (≤ 64
// columns × m rows) for the whole solve, so a pass is a local shared-memory product; everything
// that is a sum over columns (the ∇ψ vector A_J P_J, the four K1 scalar partials, |J|) leaves each
// CTA as one record and is combined by EVERY CTA from the 16 records in rank order (bitwise the
// same sums everywhere), so the control decisions of Algorithm 1 — inner/outer stops (R6, R7),
// Armijo with the roundoff guard (R29), halving (R5), stall (R30), factor retry (R36), the R37
// schedule, σ ← min(5σ, σmax) — are taken redundantly and identically by all CTAs with no
// broadcast.  Newton systems (Eq. (18)/(19)): the entries of the (r+1) × r (SMW, with u = A_Jᵀg as
// row r) or (m+1) × m (rhs g as row m) matrix are split over the 16 CTAs, each computes its share
// in a fixed order and stores it into every CTA's copy (DSMEM stores), one cluster barrier, then
// every CTA factors the identical matrix (blocked by 8 columns: one warp factors the panel in
// registers, all warps apply the rank-8 update) and solves for the identical d.
//
// Operation order follows the one-CTA path / the oracle where the oracle fixes it (prox, Armijo,
// σ update, res1/res3 formulas, branch rule); reduction orders differ, so results agree with the
// other paths and the oracle up to rounding (the tests compare against the oracle).
#pragma once
#include <cooperative_groups.h>

#include "k_small.cuh"

namespace ssn {

#ifdef SMALL_PROF  // phase cycle totals of rank 0 / thread 0 (same counters as k_small_solve):
// pass, local epilogue + ∇ψ partial, record exchange, Newton matrix, factor, bwd + d + gᵀd, gradient
#define CPROF_T0() long long cp_t0_ = clock64()
#define CPROF_ADD(k) do { if (q == 0 && tid == 0) { const long long t_ = clock64(); g_small_prof[k] += t_ - cp_t0_; cp_t0_ = t_; } } while (0)
#else
#define CPROF_T0() do {} while (0)
#define CPROF_ADD(k) do {} while (0)
#endif

constexpr int kClCtas = 16;
constexpr int kClThreads = 256;
constexpr int kClNW = kClThreads / 32;
constexpr int kClCols = kSmallMaxN / kClCtas;  // ≤ 64 columns per CTA
constexpr int kClLd = kSmallMaxM + 2;          // Newton matrix leading dimension (≤ 65 rows)
constexpr int kClRec = kSmallMaxM + 8;         // record: ∇ψ partial (64) | 4 scalar partials | count
constexpr int kClE = (kSmallMaxM + 1) * (kSmallMaxM + 2) / 2;  // ≥ lower-triangle entries + rhs row

// shared-memory layout (doubles)
constexpr int kClOffAs = 0;                                        // A block: column a at a·m
constexpr int kClOffW = kClOffAs + kClCols * kSmallMaxM;           // w[3][64]
constexpr int kClOffX = kClOffW + 3 * kClCols;                     // x (local)
constexpr int kClOffPl = kClOffX + kClCols;                        // P_J local [2][64]
constexpr int kClOffY = kClOffPl + 2 * kClCols;                    // y[2][64]
constexpr int kClOffG = kClOffY + 2 * kSmallMaxM;                  // g[2][64]
constexpr int kClOffD = kClOffG + 2 * kSmallMaxM;                  // d, b, v, Gsum
constexpr int kClOffRec = kClOffD + 4 * kSmallMaxM;                // records [2][kClRec]
constexpr int kClOffAJ = kClOffRec + 2 * kClRec;                   // gathered A_J / local partial Gram
constexpr int kClOffM = kClOffAJ + kSmallMaxM * kSmallMaxM;        // Newton matrix [65][66]
constexpr int kClLpLd = 72;                                        // panel L, transposed: Lp[p·72 + i]
constexpr int kClOffLp = kClOffM + (kSmallMaxM + 1) * kClLd;
constexpr int kClOffLd = kClOffLp + 8 * kClLpLd;                   // diag L, 1/diag [2][64]
constexpr int kClOffRed = kClOffLd + 2 * kSmallMaxM;               // scalar partials [8] + per-part rows [4][64]
constexpr int kClOffSc = kClOffRed + 5 * kSmallMaxM;               // scalars
constexpr int kClDoubles = kClOffSc + 64;
constexpr size_t kClSmem = (size_t)8 * kClDoubles + (size_t)4 * (2 * kClCols + 2 * kSmallMaxM + 48 + 8);

__global__ void __cluster_dims__(kClCtas, 1, 1) __launch_bounds__(kClThreads, 1) k_small_cl(const SmallParams p) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) double sm[];
  const int m = p.m, n = p.n;
  const int q = (int)cluster.block_rank();
  const int c0 = (int)((int64_t)n * q / kClCtas), c1 = (int)((int64_t)n * (q + 1) / kClCtas);
  const int nl = c1 - c0;
  double* As = sm + kClOffAs;
  double* w = sm + kClOffW;  // w[c] = w + c·kClCols
  double* xs = sm + kClOffX;
  double* Pl = sm + kClOffPl;  // Pl[c] = Pl + c·kClCols
  double* ys = sm + kClOffY;
  double* gs = sm + kClOffG;
  double* ds = sm + kClOffD;
  double* bs = ds + kSmallMaxM;
  double* vs = bs + kSmallMaxM;
  double* Gs = vs + kSmallMaxM;  // Σ_ranks ∇ψ partial
  double* rec = sm + kClOffRec;
  double* AJ = sm + kClOffAJ;
  double* Mx = sm + kClOffM;
  double* Lp = sm + kClOffLp;
  double* Ld = sm + kClOffLd;
  double* red = sm + kClOffRed;
  double* sc_ = sm + kClOffSc;
  int* Jl = (int*)(sm + kClDoubles);       // Jl[c] = Jl + c·kClCols (local column indices, ascending)
  int* Jg = Jl + 2 * kClCols;              // gathered: (rank << 8) | local column, per global J position
  int* offsb = Jg + 2 * kSmallMaxM;        // offsb[jc·17 + q]: exclusive prefix of the ranks' |J[jc]| counts
  int* iscr = offsb + 48;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr unsigned FULL = 0xffffffffu;

  __shared__ DevCtl C;
  if (tid == 0) {
    C = p.use_cin ? p.cin : *p.C;
    if (p.sigma_in) C.sigma = *p.sigma_in;  // σ0 carried from the previous path point (R38)
  }
  for (int e = tid; e < nl * m; e += kClThreads) As[e] = __ldg(p.A + (int64_t)c0 * m + e);
  for (int i = tid; i < nl; i += kClThreads) {  // cold start (R8): x = 0, y0 = 0, w0 = Aᵀ0 = 0
    xs[i] = p.cold ? 0.0 : p.x[c0 + i];
    w[i] = p.cold ? 0.0 : p.w0[c0 + i];
  }
  if (tid < m) {
    ys[tid] = p.cold ? 0.0 : p.y0[tid];
    bs[tid] = p.b[tid];
  }
  if (p.cold && q == 0 && tid == 0) {
    *p.rx0 = 0;
    if (p.rx0_host) *reinterpret_cast<int64_t*>(p.rx0_host) = 0;
  }
  __syncthreads();
  const double l1 = C.l1, l2 = C.l2, tol = C.tol, nb = C.nb;
  int rbuf = 0;  // record buffer parity (see exchange)

  // w_dst (local) = A_blockᵀ y: thread t → column t/4, rows ≡ t (mod 4), two xor shuffles (fixed order)
  auto pass = [&](const double* yv, double* wdst) {
    CPROF_T0();
    const int a = tid >> 2, part = tid & 3;
    double s0 = 0.0, s1 = 0.0;
    if (a < nl) {
      const double* col = As + a * m;
      int k = part;
      for (; k + 4 < m; k += 8) {
        s0 = __fma_rn(col[k], yv[k], s0);
        s1 = __fma_rn(col[k + 4], yv[k + 4], s1);
      }
      if (k < m) s0 = __fma_rn(col[k], yv[k], s0);
    }
    double v = __dadd_rn(s0, s1);
    v = __dadd_rn(v, __shfl_xor_sync(FULL, v, 1));
    v = __dadd_rn(v, __shfl_xor_sync(FULL, v, 2));
    if (part == 0 && a < nl) wdst[a] = v;
    __syncthreads();
    CPROF_ADD(0);
  };

  // Local epilogue (threads 0..63, one column each): w_eff = w0 (+ step (w1 − w0)) [→ wout], t = x − σw,
  // P, ordered local compaction → (Jl[jc], Pl[jc]), scalar partials; then (with_grad) the local
  // ∇ψ partial Σ_{a ∈ J_q} P_a a_a; the record goes to rec[rbuf] and every CTA combines the 16
  // records in rank order: Gs, S[4] (sc_[0..3]), offsets, r.  Returns r (global |J|).
  auto evaluate = [&](const Scal& sc, const double* w0p, const double* w1p, double step, double* wout, int jc,
                      bool with_grad) -> int {
    CPROF_T0();
    double s[4] = {0, 0, 0, 0};
    double P = 0.0;
    int act = 0;
    if (tid < kClCols) {
      const int a = tid;
      if (a < nl) {
        double ww = w0p[a];
        if (w1p) ww = __dadd_rn(ww, __dmul_rn(step, __dsub_rn(w1p[a], ww)));
        if (wout) wout[a] = ww;
        const double xi = xs[a];
        const double tt = __dsub_rn(xi, __dmul_rn(sc.sigma, ww));
        act = fabs(tt) > sc.thr;
        P = prox_en(tt, sc.thr, sc.den);
        const double dx = __dsub_rn(xi, P);
        const double z = __dsub_rn(__ddiv_rn(dx, sc.sigma), ww);
        const double e = __dsub_rn(fabs(ww), sc.l1);
        s[0] = __dmul_rn(P, P);
        s[1] = __dmul_rn(dx, dx);
        s[2] = __dmul_rn(z, z);
        s[3] = e > 0.0 ? __dmul_rn(e, e) : 0.0;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) s[j] = warp_allsum(s[j]);
      const unsigned bal = __ballot_sync(FULL, act);
      if (lane == 0) {
        iscr[warp] = __popc(bal);
        for (int j = 0; j < 4; ++j) red[warp * 4 + j] = s[j];
      }
      named_bar_sync(1, kClCols);
      const int pos = (warp ? iscr[0] : 0) + __popc(bal & lanemask_lt());
      if (act) {
        Jl[jc * kClCols + pos] = a;
        Pl[jc * kClCols + pos] = P;
      }
    }
    __syncthreads();
    const int cnt = iscr[0] + (kClCols > 32 ? iscr[1] : 0);
    double* R = rec + rbuf * kClRec;
    if (with_grad) {  // thread (k, part): Σ over a ≡ part (mod 4) of P_a A[k, J_a]
      const int k = tid & 63, part = tid >> 6;
      double acc = 0.0;
      if (k < m)
        for (int a = part; a < cnt; a += 4)
          acc = __fma_rn(Pl[jc * kClCols + a], As[Jl[jc * kClCols + a] * m + k], acc);
      red[32 + part * 64 + k] = acc;  // red[32 ..) free: the scalar partials use red[0 .. 8)
    }
    __syncthreads();
    if (tid < kSmallMaxM) {
      double v = 0.0;
      if (with_grad && tid < m)
        v = __dadd_rn(__dadd_rn(red[32 + tid], red[32 + 64 + tid]), __dadd_rn(red[32 + 128 + tid], red[32 + 192 + tid]));
      R[tid] = v;
    }
    if (tid < 4) R[kSmallMaxM + tid] = __dadd_rn(red[tid], red[4 + tid]);
    if (tid == 4) R[kSmallMaxM + 4] = (double)cnt;
    CPROF_ADD(1);
    cluster.sync();  // records of all ranks visible
    if (tid < m) {
      double v = 0.0;
      for (int rq = 0; rq < kClCtas; ++rq) v = __dadd_rn(v, cluster.map_shared_rank(R, rq)[tid]);
      Gs[tid] = v;
    } else if (tid >= 64 && tid < 68) {
      double v = 0.0;
      for (int rq = 0; rq < kClCtas; ++rq) v = __dadd_rn(v, cluster.map_shared_rank(R, rq)[kSmallMaxM + tid - 64]);
      sc_[tid - 64] = v;
    } else if (tid == 96) {
      int* offs = offsb + jc * (kClCtas + 1);
      int o = 0;
      for (int rq = 0; rq < kClCtas; ++rq) {
        offs[rq] = o;
        o += (int)cluster.map_shared_rank(R, rq)[kSmallMaxM + 4];
      }
      offs[kClCtas] = o;
    }
    __syncthreads();
    CPROF_ADD(2);
    rbuf ^= 1;  // the next record goes to the other buffer: a rank rewrites this one only after the
                // next cluster barrier, i.e. after every rank has finished reading it
    return offsb[jc * (kClCtas + 1) + kClCtas];
  };

  // g = y + b − Gs (with_grad) and (yy, by, gg) → out[0..2]; identical on every CTA
  auto gradient = [&](const double* yv, double* gdst, double (&out)[3], bool with_grad) {
    CPROF_T0();
    if (warp == 0) {
      double yy = 0.0, by = 0.0, gg = 0.0;
      for (int h = 0; h < 2; ++h) {
        const int k = lane + 32 * h;
        if (k < m) {
          const double yk = yv[k], bk = bs[k];
          yy = __dadd_rn(yy, __dmul_rn(yk, yk));
          by = __dadd_rn(by, __dmul_rn(bk, yk));
          if (with_grad) {
            const double g = __dsub_rn(__dadd_rn(yk, bk), Gs[k]);
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
    CPROF_ADD(6);
  };

  auto make_ev = [&](const Scal& sc, const double (&q3)[3], int r, bool with_grad) {
    EvalOut o;
    o.yy = q3[0];
    o.by = q3[1];
    o.gg = q3[2];
    for (int j = 0; j < 4; ++j) o.s[j] = sc_[j];
    const double tprox = __dmul_rn(sc.cpsi, o.s[0]);
    o.psi = __dadd_rn(__dadd_rn(__dmul_rn(0.5, q3[0]), q3[1]), tprox);
    o.psimag = fabs(0.5 * q3[0]) + fabs(q3[1]) + fabs(tprox);
    o.res1 = with_grad ? sqrt(q3[2]) / (1.0 + nb) : -1.0;
    o.gd = 0.0;
    o.r = r;
    o.info = 0;
    o.seq = 0;
    o.pad = 0;
    return o;
  };

  // Newton direction at (g = gs[cur], J[cur], r): d (ds), gᵀd, branch; false on a bad pivot.
  auto direction = [&](int cur, int r, double kappa, double jit, double& gd, int& br) -> bool {
    const double* g = gs + cur * kSmallMaxM;
    const int* offs = offsb + cur * (kClCtas + 1);  // the rank offsets of THIS set (a retry follows a trial)
    CPROF_T0();
    if (r == 0) {
      br = 0;
      if (tid < m) ds[tid] = -g[tid];
    } else {
      const bool smw = r < m;
      br = smw ? 1 : 2;
      const int N = smw ? r : m;
      // Matrix entries (i, c), i ≥ c (rows i ≤ N: row N is the right-hand side): rank q computes the
      // columns c ≡ q (mod 16), warp per column, lanes over rows, and stores them into every rank's copy.
      if (smw) {
        // gather the r active columns (position j = offs[rank] + local index): warp w takes positions
        // j ≡ w (mod 8); the owner's local index and the column rows arrive in two DSMEM round trips
        for (int j0 = warp; j0 < r; j0 += 8 * kClNW) {
          int code = 0;
          if (lane < 8 && j0 + kClNW * lane < r) {
            const int j = j0 + kClNW * lane;
            int rq = 0;
            while (rq + 1 < kClCtas && offs[rq + 1] <= j) ++rq;
            code = (rq << 8) | cluster.map_shared_rank(Jl + cur * kClCols, rq)[j - offs[rq]];
          }
          double vals[8][2];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int cu = __shfl_sync(FULL, code, u);
            const int j = j0 + kClNW * u;
            const double* src = cluster.map_shared_rank(As, cu >> 8) + (cu & 255) * m;
            vals[u][0] = (j < r && lane < m) ? src[lane] : 0.0;
            vals[u][1] = (j < r && lane + 32 < m) ? src[lane + 32] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int j = j0 + kClNW * u;
            if (j < r) {
              if (lane < m) AJ[j * m + lane] = vals[u][0];
              if (lane + 32 < m) AJ[j * m + lane + 32] = vals[u][1];
            }
          }
        }
        __syncthreads();
        // κ⁻¹I_r + A_JᵀA_J (lower) and u = A_Jᵀg (row N)
        for (int c = q + kClCtas * warp; c < N; c += kClCtas * kClNW) {
          const double* bc = AJ + c * m;
          for (int i = c + lane; i <= N; i += 32) {
            const double* ai = i < N ? AJ + i * m : g;
            double s0 = 0.0, s1 = 0.0;
            int k = 0;
            for (; k + 1 < m; k += 2) {
              s0 = __fma_rn(ai[k], bc[k], s0);
              s1 = __fma_rn(ai[k + 1], bc[k + 1], s1);
            }
            if (k < m) s0 = __fma_rn(ai[k], bc[k], s0);
            double v = __dadd_rn(s0, s1);
            if (i == c) {
              v = __dadd_rn(v, 1.0 / kappa);
              if (jit != 0.0) v = __fma_rn(v, jit, v);
            }
            for (int rq = 0; rq < kClCtas; ++rq) cluster.map_shared_rank(Mx, rq)[i + c * kClLd] = v;
          }
        }
      } else {
        // local partial Gram Σ_{a ∈ J_q} a_a a_aᵀ (lower m × m, AJ[i + 64 c]), then this rank's columns of
        // I_m + κ Σ_ranks (partials), the partials summed in rank order, into every rank's copy
        const int cnt = offs[q + 1] - offs[q];
        const int* Jc = Jl + cur * kClCols;
        for (int c = warp; c < m; c += kClNW)
          for (int i = c + lane; i < m; i += 32) {
            double s0 = 0.0, s1 = 0.0;
            int a = 0;
            for (; a + 1 < cnt; a += 2) {
              const double* c0p = As + Jc[a] * m;
              const double* c1p = As + Jc[a + 1] * m;
              s0 = __fma_rn(c0p[i], c0p[c], s0);
              s1 = __fma_rn(c1p[i], c1p[c], s1);
            }
            if (a < cnt) s0 = __fma_rn(As[Jc[a] * m + i], As[Jc[a] * m + c], s0);
            AJ[i + kSmallMaxM * c] = __dadd_rn(s0, s1);
          }
        cluster.sync();  // every rank's partial Gram complete
        for (int c = q + kClCtas * warp; c < m; c += kClCtas * kClNW)
          for (int i = c + lane; i < m; i += 32) {
            double sv[kClCtas];
#pragma unroll
            for (int rq = 0; rq < kClCtas; ++rq) sv[rq] = cluster.map_shared_rank(AJ, rq)[i + kSmallMaxM * c];
            double s = 0.0;
#pragma unroll
            for (int rq = 0; rq < kClCtas; ++rq) s = __dadd_rn(s, sv[rq]);
            double v = __dadd_rn(__dmul_rn(kappa, s), i == c ? 1.0 : 0.0);
            if (i == c && jit != 0.0) v = __fma_rn(v, jit, v);
            for (int rq = 0; rq < kClCtas; ++rq) cluster.map_shared_rank(Mx, rq)[i + c * kClLd] = v;
          }
        if (tid < m) Mx[m + tid * kClLd] = g[tid];
      }
      cluster.sync();  // every copy of the Newton matrix complete (and the partial Grams read)
      CPROF_ADD(3);
#ifdef SMALL_PROF
      if (q == 0 && tid == 0) g_small_prof[6] += (unsigned long long)N << 32;  // Σ N in the high half
#endif

      // ---- Cholesky with the rhs as row N (forward substitution for free), blocked by 8 columns:
      // warp 0 factors the 8-column panel (rows jb … N) in registers; L[i][j] (i > j, incl. row N)
      // goes to the upper triangle Mx[j + i·ld] and to the panel buffer Lp[p·72 + i]; then every warp
      // applies the rank-8 update to the trailing lower triangle (incl. row N): warp w takes columns
      // c ≡ w (mod 8), lanes take rows (consecutive rows: conflict-free shared-memory access).
      int badl = 0;
      for (int jb = 0; jb < N; jb += 8) {
        const int nbk = min(8, N - jb);
        if (warp == 0) {
          // as diag_factor4 (k_newton.cuh): every lane keeps a replica of the 8 panel diagonals and
          // updates it from the shuffled L values, so each pivot is local (one shuffle per pivot on the
          // chain); pivots past the matrix are padded (d = 1, zero column), so no shuffle is conditional
          double v[3][8], dg[8];
#pragma unroll
          for (int h = 0; h < 3; ++h) {
            const int i = jb + lane + 32 * h;
#pragma unroll
            for (int pp = 0; pp < 8; ++pp) v[h][pp] = (i <= N && pp < nbk) ? Mx[i + (jb + pp) * kClLd] : 0.0;
          }
#pragma unroll
          for (int pp = 0; pp < 8; ++pp) dg[pp] = pp < nbk ? Mx[(jb + pp) * (kClLd + 1)] : 1.0;
#pragma unroll
          for (int pp = 0; pp < 8; ++pp) {
            const double dd = dg[pp];
            const bool ok = dd > 0.0;
            badl |= (pp < nbk) && !ok;
            const double dv = ok ? dd : 1.0;
            const double inv = rsqrt_pos(dv);
#pragma unroll
            for (int h = 0; h < 3; ++h) {
              const int i = jb + lane + 32 * h;
              v[h][pp] = i > jb + pp ? __dmul_rn(v[h][pp], inv) : 0.0;
            }
#pragma unroll
            for (int qq = pp + 1; qq < 8; ++qq) {
              const double lq = __shfl_sync(FULL, v[0][pp], qq);  // L[jb + qq][jb + pp] (0 past the matrix)
              dg[qq] = __fma_rn(-lq, lq, dg[qq]);
#pragma unroll
              for (int h = 0; h < 3; ++h) v[h][qq] = __fma_rn(-v[h][pp], lq, v[h][qq]);
            }
            if (lane == 0 && pp < nbk) {
              Ld[jb + pp] = __dmul_rn(dv, inv);
              Ld[kSmallMaxM + jb + pp] = inv;
            }
          }
#pragma unroll
          for (int h = 0; h < 3; ++h) {
            const int i = jb + lane + 32 * h;
            if (i <= N)
#pragma unroll
              for (int pp = 0; pp < 8; ++pp)
                if (pp < nbk && i > jb + pp) {
                  Mx[(jb + pp) + i * kClLd] = v[h][pp];
                  Lp[pp * kClLpLd + i] = v[h][pp];
                }
          }
        }
        __syncthreads();
        CPROF_ADD(7);
        const int j1 = jb + nbk;
        for (int c = j1 + warp; c < N; c += kClNW) {
          double lc[8];
#pragma unroll
          for (int pp = 0; pp < 8; ++pp) lc[pp] = pp < nbk ? Lp[pp * kClLpLd + c] : 0.0;  // broadcast
          for (int i = c + lane; i <= N; i += 32) {
            double acc = Mx[i + c * kClLd];
#pragma unroll
            for (int pp = 0; pp < 8; ++pp)
              if (pp < nbk) acc = __fma_rn(-Lp[pp * kClLpLd + i], lc[pp], acc);
            Mx[i + c * kClLd] = acc;
          }
        }
        __syncthreads();
        CPROF_ADD(4);
      }
      if (warp == 0) {
        badl = __any_sync(FULL, badl);
        if (lane == 0) sc_[16] = badl ? 1.0 : 0.0;
      }
      __syncthreads();
      CPROF_ADD(4);
      const int bad = sc_[16] != 0.0;
      // ---- backward substitution v = L⁻ᵀ z (z = row N), one warp; rows lane and lane + 32 ----
      if (warp == 0) {
        double z0 = lane < N ? Mx[lane + N * kClLd] : 0.0, z1 = lane + 32 < N ? Mx[lane + 32 + N * kClLd] : 0.0;
        for (int i = N - 1; i >= 0; --i) {
          const double zi = __shfl_sync(FULL, i < 32 ? z0 : z1, i & 31);
          const double vi = __dmul_rn(zi, Ld[kSmallMaxM + i]);
          if (lane == (i & 31)) {
            if (i < 32) z0 = vi;
            else z1 = vi;
          }
          if (lane < i) z0 = __fma_rn(-Mx[lane + i * kClLd], vi, z0);
          if (lane + 32 < i) z1 = __fma_rn(-Mx[lane + 32 + i * kClLd], vi, z1);
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
    CPROF_ADD(5);
    return true;
  };

  // ---- Algorithm 1 (same control flow as k_small_solve) ----
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
    double q3[3];
    r_cur = evaluate(sc, w + wcur * kClCols, nullptr, 0.0, nullptr, cur, true);
    gradient(ys + cur * kSmallMaxM, gs + cur * kSmallMaxM, q3, true);
    ev = make_ev(sc, q3, r_cur, true);
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
      const bool fok = direction(cur, r_cur, sc.kappa, retry ? C.jitter : 0.0, gd, br);
      brs[br]++;
      if (tid < m) ys[tr * kSmallMaxM + tid] = __dadd_rn(ys[cur * kSmallMaxM + tid], ds[tid]);
      __syncthreads();
      pass(ys + tr * kSmallMaxM, w + wtr * kClCols);
      aty++;
      double qt3[3];
      const int r_t = evaluate(sc, w + wtr * kClCols, nullptr, 0.0, nullptr, tr, true);
      gradient(ys + tr * kSmallMaxM, gs + tr * kSmallMaxM, qt3, true);
      EvalOut evt = make_ev(sc, qt3, r_t, true);
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
        double qb3[3];
        const int r_b = evaluate(sc, w + wcur * kClCols, w + wtr * kClCols, s, w + wbt * kClCols, tr, false);
        gradient(ys + tr * kSmallMaxM, nullptr, qb3, false);
        evt = make_ev(sc, qb3, r_b, false);
        psi_evals++;
        ok = armijo(evt.psi);
      }
      backtracks += nbt;
      if (nbt == 0) {
        cur = tr;
        wcur = wtr;
        ev = evt;
        r_cur = r_t;
      } else {  // the accepted point needs ∇ψ for its re-thresholded J: recompute the local partials
        cur = tr;
        wcur = wbt;
        double q2[3];
        r_cur = evaluate(sc, w + wcur * kClCols, nullptr, 0.0, nullptr, cur, true);
        gradient(ys + cur * kSmallMaxM, gs + cur * kSmallMaxM, q2, true);
        ev = make_ev(sc, q2, r_cur, true);
      }
      newton++;
      retry = 0;
    }
    if (numeric) break;
    res3 = (sqrt(ev.s[1]) / sigma) / (1.0 + sqrt(ev.yy) + sqrt(ev.s[2]));
    res1 = ev.res1;
    // multiplier update Eq. (10): x ← P, local columns; support list at the rank's offset.
    // The current dual iterate (y, w = Aᵀy) goes to y0 / w0 at every outer step: the last one is the
    // final iterate the next point of a path starts from (reading R39; every CTA read y0 / w0 at the
    // start, before the first cluster barrier)
    const int* offs = offsb + cur * (kClCtas + 1);
    const int cntq = offs[q + 1] - offs[q];
    for (int i = tid; i < nl; i += kClThreads) {
      xs[i] = 0.0;
      p.w0[c0 + i] = w[wcur * kClCols + i];
    }
    if (q == 0 && tid < m) p.y0[tid] = ys[cur * kSmallMaxM + tid];
    __syncthreads();
    for (int a = tid; a < cntq; a += kClThreads) {
      const int la = Jl[cur * kClCols + a];
      const double v = Pl[cur * kClCols + a];
      xs[la] = v;
      p.Jx[offs[q] + a] = c0 + la;
      p.Px[offs[q] + a] = v;
    }
    if (q == 0 && tid == 0) *p.rx = r_cur;
    __syncthreads();
    if (res3 <= tol && ev.res1 <= tol) {
      converged = 1;
      k++;
      break;
    }
    sigma = fmin(C.sigma_factor * sigma, C.sigma_max);
  }
  // ---- objective pieces of the final x (Eq. (1)): A x from the local dense x, one more record
  // exchange (rank order), then rank 0 forms ½‖Ax − b‖², Σ|x|, Σx², nnz and A x − b ----
  if (p.obj) {
    double* R = rec + rbuf * kClRec;
    {
      const int k = tid & 63, part = tid >> 6;
      double acc = 0.0;
      if (k < m)
        for (int a = part; a < nl; a += 4)
          if (xs[a] != 0.0) acc = __fma_rn(xs[a], As[a * m + k], acc);
      red[32 + part * 64 + k] = acc;
    }
    if (warp == 7) {
      double l1s = 0.0, l2s = 0.0, nz = 0.0;
      for (int a = lane; a < nl; a += 32) {
        const double xv = xs[a];
        l1s = __dadd_rn(l1s, fabs(xv));
        l2s = __dadd_rn(l2s, __dmul_rn(xv, xv));
        nz += xv != 0.0 ? 1.0 : 0.0;
      }
      l1s = warp_allsum(l1s);
      l2s = warp_allsum(l2s);
      nz = warp_allsum(nz);
      if (lane == 0) {
        R[kSmallMaxM] = l1s;
        R[kSmallMaxM + 1] = l2s;
        R[kSmallMaxM + 2] = nz;
      }
    }
    __syncthreads();
    if (tid < m)
      R[tid] = __dadd_rn(__dadd_rn(red[32 + tid], red[32 + 64 + tid]), __dadd_rn(red[32 + 128 + tid], red[32 + 192 + tid]));
    cluster.sync();
    if (q == 0) {
      if (warp == 0) {
        double rr = 0.0;
        for (int h = 0; h < 2; ++h) {
          const int k = lane + 32 * h;
          if (k < m) {
            double v = 0.0;
            for (int rq = 0; rq < kClCtas; ++rq) v = __dadd_rn(v, cluster.map_shared_rank(R, rq)[k]);
            const double res = __dsub_rn(v, bs[k]);
            if (p.resid) p.resid[k] = res;
            rr = __dadd_rn(rr, __dmul_rn(res, res));
          }
        }
        rr = warp_allsum(rr);
        if (lane == 0) p.obj[0] = 0.5 * rr;
      } else if (tid == 32) {
        double t3[3] = {0.0, 0.0, 0.0};
        for (int rq = 0; rq < kClCtas; ++rq)
          for (int j = 0; j < 3; ++j) t3[j] = __dadd_rn(t3[j], cluster.map_shared_rank(R, rq)[kSmallMaxM + j]);
        p.obj[1] = t3[0];
        p.obj[2] = t3[1];
        p.obj[3] = t3[2];
      }
    }
  }
  // ---- outputs ----
  for (int i = tid; i < nl; i += kClThreads) {
    p.x[c0 + i] = xs[i];
    if (p.xout) p.xout[c0 + i] = xs[i];
  }
  if (q == 0 && tid == 0) {
    DevCtl o = C;  // settings as used, then the statistics
    o.outer_iters = k;
    o.newton_iters = newton;
    o.psi_evals = psi_evals;
    o.backtracks = backtracks;
    o.aty_passes = aty;
    for (int b = 0; b < 4; ++b) o.branch_steps[b] = brs[b];
    o.cg_iters = 0;
    o.jitter_retries = jretries;
    o.stalled = stalled;
    o.res1 = res1;
    o.res3 = res3;
    o.sigma_final = sigma;
    o.converged = converged;
    o.numeric = numeric;
    o.numeric_kind = numeric_kind;
    o.numeric_r = numeric_r;
    o.seg_outer = o.seg_inner = o.seg_bt = o.seg_grad = 0;
    o.k1_ns = 0;
    o.k1_cnt = 0;
    *p.C = o;  // device control block (the carried σ of a path is read from it)
    *p.ev = ev;
    if (p.cout_host) *p.cout_host = o;  // the mapped host mirrors: no copies after the launch
    if (p.ev_host) *p.ev_host = ev;
  }
  cluster.sync();  // no rank exits while another may still read its shared memory
}

}  // namespace ssn
