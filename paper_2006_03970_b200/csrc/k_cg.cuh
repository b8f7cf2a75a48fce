// k_cg.cuh — K6: the Newton direction by conjugate gradient (Algorithm 1 step (1): "solving
// exactly or by conjugate gradient"), matrix-free: V u = u + κ A_J (A_Jᵀ u).
//
// One cooperative launch runs the whole CG loop (reading R32: d0 = 0, stop at
// ‖V d + g‖ ≤ tol·‖g‖ or maxit), persistent CTAs with two grid barriers per iteration:
//   phase 1  each CTA owns a contiguous range of J; warp w takes columns a ≡ w (mod 8) of it:
//            t_a = a_aᵀ p (column in registers, butterfly dot), then the warp's partial
//            Σ t_a a_a from the same registers (A_J is read once per iteration) and Σ t_a².
//            CTA partials (warps in order) → parts[b], tts[b].                    | grid sync
//   phase 2  every CTA: pᵀVp = pᵀp + κ Σ_b tts[b]  (b ascending), α = rr / pᵀVp; on its row
//            slice q = p + κ Σ_b parts[b] (b ascending), d += α p, res −= α q, Σ res² → rrs[b]
//                                                                                    | grid sync
//   phase 3  every CTA redundantly: rr' = Σ_b rrs[b], β = rr'/rr, p = res + β p (full m in
//            smem, identical in all CTAs), pᵀp in a fixed order.
// Every reduction has a fixed order: results do not depend on timing.  The last CTA-0 step
// writes gᵀd and the Armijo trial y + d like the direct branches.
#pragma once
#include <cooperative_groups.h>
#include "common.cuh"
#include "k_newton.cuh"

namespace ssn {

constexpr int K6_THREADS = 256;

struct CgParams {
  int64_t m;
  const int32_t* J;
  int64_t r;            // overridden by geo
  const double* g;
  double kappa;         // overridden by geo (mult)
  double tol;
  int maxit;
  const double* y;      // Armijo base point (nullable)
  double* d;            // m: solution
  double* yt;           // m: y + d (nullable)
  double* gd_out;       // gᵀd
  double* res;          // m scratch: residual −g − V d
  double* parts;        // gridDim × m
  double* scal;         // gridDim × 2: [tt, rr] partials
  int* iters_out;       // += iterations (nullable)
  const DirGeo* geo;    // graph mode: branch 3 predicate, r, κ
};

// deterministic block sum of one double per thread (all threads get the result)
SSN_DEV double block_sum(double v, double* red, int tid) {
  v = warp_allsum(v);
  __syncthreads();
  if ((tid & 31) == 0) red[tid >> 5] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < K6_THREADS / 32; ++w) s += red[w];
  return s;
}

template <class Acc, int MR>
__global__ void __launch_bounds__(K6_THREADS, 1) k_cg_newton(const CgParams prm, const Acc A) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  int64_t r = prm.r;
  double kappa = prm.kappa;
  if (prm.geo) {
    if (prm.geo->branch != 3) return;  // uniform over the grid
    r = prm.geo->r;
    kappa = prm.geo->mult;
  }
  extern __shared__ double sm[];
  const int64_t m = prm.m;
  double* p = sm;                         // m
  double* wpart = sm + ((m + 31) / 32) * 32;  // 8 × m warp partials
  __shared__ double red[K6_THREADS / 32];
  __shared__ double wtt[K6_THREADS / 32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int b = blockIdx.x, G = gridDim.x;
  const int64_t a_lo = (int64_t)b * r / G, a_hi = (int64_t)(b + 1) * r / G;
  const int64_t k_lo = (int64_t)b * m / G, k_hi = (int64_t)(b + 1) * m / G;
  // ---- setup: d = 0, res = −g, p = −g, rr = gᵀg (every CTA, same order) ----
  double gg_l = 0.0;
  for (int64_t k = tid; k < m; k += K6_THREADS) {
    const double gk = prm.g[k];
    p[k] = -gk;
    gg_l += gk * gk;
  }
  for (int64_t k = k_lo + tid; k < k_hi; k += K6_THREADS) {
    prm.d[k] = 0.0;
    prm.res[k] = -prm.g[k];
  }
  const double gg = block_sum(gg_l, red, tid);
  double rr = gg, pp = gg;
  const double thr = prm.tol * prm.tol * gg;
  int it = 0;
  while (it < prm.maxit && rr > thr) {  // uniform: every CTA holds identical rr
    // ---- phase 1: t_a = a_aᵀ p, warp partial Σ t_a a_a, Σ t_a² ----
    double pr[MR], acc[MR];
#pragma unroll
    for (int t = 0; t < MR; ++t) {
      const int64_t row = lane + 32 * t;
      pr[t] = row < m ? p[row] : 0.0;
      acc[t] = 0.0;
    }
    double tt = 0.0;
    for (int64_t a = a_lo + warp; a < a_hi; a += 8) {
      const auto col = A.col(prm.J[a]);
      double cv[MR];
      double s = 0.0;
#pragma unroll
      for (int t = 0; t < MR; ++t) {
        const int64_t row = lane + 32 * t;
        cv[t] = row < m ? col.ld(row) : 0.0;
        s = fma(cv[t], pr[t], s);
      }
      s = warp_allsum(s);  // t_a (bitwise identical in all lanes)
      tt = fma(s, s, tt);
#pragma unroll
      for (int t = 0; t < MR; ++t) acc[t] = fma(s, cv[t], acc[t]);
    }
#pragma unroll
    for (int t = 0; t < MR; ++t) {
      const int64_t row = lane + 32 * t;
      if (row < m) wpart[(size_t)warp * m + row] = acc[t];
    }
    if (lane == 0) wtt[warp] = tt;
    __syncthreads();
    for (int64_t k = tid; k < m; k += K6_THREADS) {
      double v = wpart[k];
      for (int w = 1; w < 8; ++w) v += wpart[(size_t)w * m + k];
      prm.parts[(size_t)b * m + k] = v;
    }
    if (tid == 0) {
      double s = wtt[0];
      for (int w = 1; w < 8; ++w) s += wtt[w];
      prm.scal[2 * b] = s;
    }
    grid.sync();
    // ---- phase 2: α, then q, d, res on this CTA's rows ----
    double ts = 0.0;
    for (int q = lane; q < G; q += 32) ts += __ldcg(prm.scal + 2 * q);
    ts = warp_allsum(ts);  // every warp computes the same value
    const double pvp = pp + kappa * ts;
    const double alpha = rr / pvp;
    double rl = 0.0;
    for (int64_t k = k_lo + tid; k < k_hi; k += K6_THREADS) {
      double s = 0.0;
      for (int q = 0; q < G; ++q) s += __ldcg(prm.parts + (size_t)q * m + k);
      const double qk = p[k] + kappa * s;
      prm.d[k] += alpha * p[k];
      const double rk = prm.res[k] - alpha * qk;
      prm.res[k] = rk;
      rl += rk * rk;
    }
    const double rb = block_sum(rl, red, tid);
    if (tid == 0) prm.scal[2 * b + 1] = rb;
    grid.sync();
    // ---- phase 3: β, p = res + β p, pᵀp (redundant in every CTA) ----
    double rs = 0.0;
    for (int q = lane; q < G; q += 32) rs += __ldcg(prm.scal + 2 * q + 1);
    const double rr_new = warp_allsum(rs);
    const double beta = rr_new / rr;
    double pl = 0.0;
    for (int64_t k = tid; k < m; k += K6_THREADS) {
      const double pk = __ldcg(prm.res + k) + beta * p[k];
      p[k] = pk;
      pl += pk * pk;
    }
    pp = block_sum(pl, red, tid);
    rr = rr_new;
    ++it;
  }
  grid.sync();  // d complete
  if (b != 0) return;
  double dl = 0.0;
  for (int64_t k = tid; k < m; k += K6_THREADS) {
    const double dk = __ldcg(prm.d + k);
    if (prm.yt) prm.yt[k] = __dadd_rn(prm.y[k], __dmul_rn(1.0, dk));
    dl += prm.g[k] * dk;
  }
  const double gd = block_sum(dl, red, tid);
  if (tid == 0) {
    *prm.gd_out = gd;
    if (prm.iters_out) *prm.iters_out += it;
  }
}

// dynamic shared memory of k_cg_newton (bytes)
inline size_t cg_smem(int64_t m) { return (size_t)(((m + 31) / 32) * 32 + 8 * m) * sizeof(double); }

}  // namespace ssn
