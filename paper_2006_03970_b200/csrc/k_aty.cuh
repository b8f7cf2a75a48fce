// k_aty.cuh — the full-width pass over A and its epilogue-only twin.
//
// K1  k1_aty_fused   : w = Aᵀy over all n columns (the only O(mn) step of a Newton
//                      iteration), fused with t = x − σw, P = prox_{σp}(t) (Eq. (6),
//                      P:170-175), the active mask |t| > σλ1 (Eq. (17)),
//                      ordered compaction of (J, P_J) into per-CTA segments, block
//                      partial sums for ψ / res3 / the dual objective, and the per-CTA
//                      m-vector Σ_{i∈J} P_i a_i used by ∇ψ (Eq. (15)).
//                      A tiles stream HBM → smem through a multi-stage ring of 1D bulk
//                      copies (cp.async.bulk, TMA) issued by one producer warp; 8 consumer
//                      warps keep y in registers (lane ℓ owns rows ℓ + 32t).
// K1e k1e_epilogue   : the same epilogue from a stored w (or w0 + s(w1 − w0) for an
//                      Armijo backtrack, by linearity of Aᵀ), no A traffic.
// K1f k1_finalize    : concatenates the per-CTA segments in CTA order → ascending J.
// K5  k_eval_reduce  : g = y + b − Σ parts, ψ (Prop. 2), res1 (Eq. (20)).
#pragma once
#include "common.cuh"

namespace ssn {

constexpr int K1_NWC = 8;                    // consumer warps
constexpr int K1_THREADS = (K1_NWC + 1) * 32; // + 1 producer warp

struct K1Params {
  const double* A;
  int64_t m, n;
  const double* y;      // m, evaluation point
  const double* x;      // n, dense multiplier (fused mode)
  double* w_out;        // n
  int32_t* seg_idx;     // n-capacity segment storage (CTA b writes from c_lo(b))
  double* seg_P;        // n
  int* cta_cnt;         // G
  double* part_scal;    // G x 4
  double* part_vec;     // G x m (fused mode; rows Σ P_i a_i)
  Scal sc;
  int C;                // columns per tile (multiple of 8)
  int64_t T;            // tiles
  int stages;
  int fused;            // 0: plain w = Aᵀy (+ max|w|), 1: full epilogue
  uint32_t stage_elems; // doubles per A stage buffer (≥ C*m, multiple of 16)
  uint32_t xstage_elems;// doubles per x stage buffer (≥ C, multiple of 16)
};

template <int MR>
__global__ void __launch_bounds__(K1_THREADS, 1) k1_aty_fused(const K1Params p) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = p.stages, C = p.C;
  const int64_t m = p.m;
  double* ring = reinterpret_cast<double*>(smem);
  double* xring = ring + (size_t)S * p.stage_elems;
  uint64_t* full = reinterpret_cast<uint64_t*>(xring + (size_t)S * p.xstage_elems);
  uint64_t* empty = full + S;
  double* wtile = reinterpret_cast<double*>(empty + S);  // 2C
  double* ptile = wtile + 2 * C;                         // 2C
  int* ftile = reinterpret_cast<int*>(ptile + 2 * C);    // 2C
  int* sh_cnt = ftile + 2 * C;

  int64_t c_lo, c_hi;
  cta_cols(blockIdx.x, gridDim.x, p.T, C, p.n, &c_lo, &c_hi);
  const int64_t ntiles = (c_hi - c_lo + C - 1) / C;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == K1_NWC) {  // ---------------- producer warp ----------------
    if (lane == 0) {
      for (int64_t it = 0; it < ntiles; ++it) {
        const int s = (int)(it % S);
        if (it >= S) mbar_wait(&empty[s], (uint32_t)(((it / S) - 1) & 1));
        const int64_t c0 = c_lo + it * C;
        const int nc = (int)((c_hi - c0) < C ? (c_hi - c0) : C);
        const uint32_t bytesA = (uint32_t)(nc * m * 8), a16 = bytesA & ~15u;
        double* dA = ring + (size_t)s * p.stage_elems;
        double* dX = xring + (size_t)s * p.xstage_elems;
        if (a16 != bytesA) dA[(size_t)nc * m - 1] = __ldg(p.A + (c0 + nc) * m - 1);  // 8-B tail
        uint32_t x16 = 0;
        if (p.fused) {
          const uint32_t bytesX = (uint32_t)nc * 8u;
          x16 = bytesX & ~15u;
          if (x16 != bytesX) dX[nc - 1] = __ldg(p.x + c0 + nc - 1);
        }
        fence_proxy_async();
        mbar_arrive_expect_tx(&full[s], a16 + x16);
        bulk_g2s(dA, p.A + c0 * m, a16, &full[s]);
        if (x16) bulk_g2s(dX, p.x + c0, x16, &full[s]);
      }
    }
    return;
  }

  // ---------------- consumer warps ----------------
  double yr[MR], gacc[MR];
#pragma unroll
  for (int t = 0; t < MR; ++t) {
    const int64_t row = lane + 32 * t;
    yr[t] = row < m ? p.y[row] : 0.0;
    gacc[t] = 0.0;
  }
  const Scal sc = p.sc;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  bool any_active = false;
  int cnt = 0;  // meaningful in warp 0

  for (int64_t it = 0; it < ntiles; ++it) {
    const int s = (int)(it % S);
    mbar_wait(&full[s], (uint32_t)((it / S) & 1));
    const int64_t c0 = c_lo + it * C;
    const int nc = (int)((c_hi - c0) < C ? (c_hi - c0) : C);
    const double* Ts = ring + (size_t)s * p.stage_elems;
    const double* Xs = xring + (size_t)s * p.xstage_elems;
    const int buf = (int)(it & 1);
    for (int c = warp; c < nc; c += K1_NWC) {
      const double* col = Ts + (size_t)c * m;
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int t = 0; t < MR; ++t) {
        const int64_t row = lane + 32 * t;
        const double v = row < m ? col[row] : 0.0;
        if (t & 1) a1 = fma(yr[t], v, a1);
        else a0 = fma(yr[t], v, a0);
      }
      const double w = warp_allsum(a0 + a1);
      if (p.fused) {
        const double xi = Xs[c];
        const double tt = __dsub_rn(xi, __dmul_rn(sc.sigma, w));
        const bool act = fabs(tt) > sc.thr;
        const double P = prox_en(tt, sc.thr, sc.den);
        const double dx = __dsub_rn(xi, P);
        const double z = __dsub_rn(__ddiv_rn(dx, sc.sigma), w);
        const double e = __dsub_rn(fabs(w), sc.l1);
        s0 = __dadd_rn(s0, __dmul_rn(P, P));
        s1 = __dadd_rn(s1, __dmul_rn(dx, dx));
        s2 = __dadd_rn(s2, __dmul_rn(z, z));
        if (e > 0.0) s3 = __dadd_rn(s3, __dmul_rn(e, e));
        if (act) {
          any_active = true;
#pragma unroll
          for (int t = 0; t < MR; ++t) {
            const int64_t row = lane + 32 * t;
            if (row < m) gacc[t] = fma(P, col[row], gacc[t]);
          }
        }
        if (lane == 0) {
          wtile[buf * C + c] = w;
          ptile[buf * C + c] = P;
          ftile[buf * C + c] = act ? 1 : 0;
        }
      } else {
        s0 = fmax(s0, fabs(w));
        if (lane == 0) wtile[buf * C + c] = w;
      }
    }
    named_bar_sync(1, K1_NWC * 32);
    if (warp == 0) {
      for (int base = 0; base < nc; base += 32) {
        const int c = base + lane;
        if (c < nc) p.w_out[c0 + c] = wtile[buf * C + c];
        if (p.fused) {
          const int f = (c < nc) ? ftile[buf * C + c] : 0;
          const unsigned bal = __ballot_sync(0xffffffffu, f);
          if (f) {
            const int pos = cnt + __popc(bal & lanemask_lt());
            p.seg_idx[c_lo + pos] = (int32_t)(c0 + c);
            p.seg_P[c_lo + pos] = ptile[buf * C + c];
          }
          cnt += __popc(bal);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }

  // ---------------- CTA reduction (fixed warp order) ----------------
  named_bar_sync(1, K1_NWC * 32);  // ring is idle now: reuse it
  double* rv = ring;                         // K1_NWC x m
  double* rs = ring + (size_t)K1_NWC * m;    // K1_NWC x 4
  int* ract = reinterpret_cast<int*>(rs + K1_NWC * 4);
  if (p.fused && p.part_vec) {
#pragma unroll
    for (int t = 0; t < MR; ++t) {
      const int64_t row = lane + 32 * t;
      if (row < m) rv[(size_t)warp * m + row] = gacc[t];
    }
  }
  if (lane == 0) {
    rs[warp * 4 + 0] = s0;
    rs[warp * 4 + 1] = s1;
    rs[warp * 4 + 2] = s2;
    rs[warp * 4 + 3] = s3;
    ract[warp] = any_active ? 1 : 0;
  }
  if (threadIdx.x == 0) *sh_cnt = cnt;
  named_bar_sync(1, K1_NWC * 32);
  const int tid = threadIdx.x;
  const int b = blockIdx.x;
  if (tid == 0) {
    double q[4] = {rs[0], rs[1], rs[2], rs[3]};
    for (int wi = 1; wi < K1_NWC; ++wi)
      for (int j = 0; j < 4; ++j) q[j] = p.fused ? __dadd_rn(q[j], rs[wi * 4 + j]) : fmax(q[j], rs[wi * 4 + j]);
    for (int j = 0; j < 4; ++j) p.part_scal[b * 4 + j] = q[j];
    p.cta_cnt[b] = p.fused ? *sh_cnt : 0;
  }
  if (p.fused && p.part_vec && *sh_cnt > 0) {
    for (int64_t k = tid; k < m; k += K1_NWC * 32) {
      double v = 0.0;
      for (int wi = 0; wi < K1_NWC; ++wi)
        if (ract[wi]) v += rv[(size_t)wi * m + k];
      p.part_vec[(size_t)b * m + k] = v;
    }
  }
}

// ---------------------------------------------------------------------------
// K1e: epilogue only.  w_eff = w0 (w1 == nullptr) or w0 + s (w1 − w0).
// ---------------------------------------------------------------------------
constexpr int K1E_THREADS = 512;

struct K1eParams {
  int64_t n;
  const double* w0;
  const double* w1;
  double s;
  const double* x;
  double* w_out;     // nullable: materialise w_eff
  int32_t* seg_idx;
  double* seg_P;
  int* cta_cnt;
  double* part_scal;
  Scal sc;
  int C;
  int64_t T;
};

__global__ void __launch_bounds__(K1E_THREADS) k1e_epilogue(const K1eParams p) {
  __shared__ int wcnt[K1E_THREADS / 32];
  __shared__ double red[K1E_THREADS / 32][4];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int64_t c_lo, c_hi;
  cta_cols(blockIdx.x, gridDim.x, p.T, p.C, p.n, &c_lo, &c_hi);
  const Scal sc = p.sc;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int64_t cnt = 0;
  for (int64_t base = c_lo; base < c_hi; base += K1E_THREADS) {
    const int64_t i = base + tid;
    int act = 0;
    double P = 0.0;
    if (i < c_hi) {
      double w = p.w0[i];
      if (p.w1) w = __dadd_rn(w, __dmul_rn(p.s, __dsub_rn(p.w1[i], w)));
      if (p.w_out) p.w_out[i] = w;
      const double xi = p.x[i];
      const double tt = __dsub_rn(xi, __dmul_rn(sc.sigma, w));
      act = fabs(tt) > sc.thr;
      P = prox_en(tt, sc.thr, sc.den);
      const double dx = __dsub_rn(xi, P);
      const double z = __dsub_rn(__ddiv_rn(dx, sc.sigma), w);
      const double e = __dsub_rn(fabs(w), sc.l1);
      s0 = __dadd_rn(s0, __dmul_rn(P, P));
      s1 = __dadd_rn(s1, __dmul_rn(dx, dx));
      s2 = __dadd_rn(s2, __dmul_rn(z, z));
      if (e > 0.0) s3 = __dadd_rn(s3, __dmul_rn(e, e));
    }
    const unsigned bal = __ballot_sync(0xffffffffu, act);
    if (lane == 0) wcnt[warp] = __popc(bal);
    __syncthreads();
    int off = 0, tot = 0;
    for (int wi = 0; wi < K1E_THREADS / 32; ++wi) {
      const int v = wcnt[wi];
      off += (wi < warp) ? v : 0;
      tot += v;
    }
    if (act) {
      const int64_t pos = cnt + off + __popc(bal & lanemask_lt());
      p.seg_idx[c_lo + pos] = (int32_t)i;
      p.seg_P[c_lo + pos] = P;
    }
    cnt += tot;
    __syncthreads();
  }
  // deterministic block reduction of the four partials
  double q[4] = {s0, s1, s2, s3};
#pragma unroll
  for (int j = 0; j < 4; ++j) q[j] = warp_allsum(q[j]);
  if (lane == 0)
    for (int j = 0; j < 4; ++j) red[warp][j] = q[j];
  __syncthreads();
  if (tid == 0) {
    double r[4] = {0, 0, 0, 0};
    for (int wi = 0; wi < K1E_THREADS / 32; ++wi)
      for (int j = 0; j < 4; ++j) r[j] += red[wi][j];
    for (int j = 0; j < 4; ++j) p.part_scal[blockIdx.x * 4 + j] = r[j];
    p.cta_cnt[blockIdx.x] = (int)cnt;
  }
}

// ---------------------------------------------------------------------------
// K1f: segments → contiguous ascending J / P_J; r → *r_out.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k1_finalize(const int32_t* __restrict__ seg_idx,
                                                   const double* __restrict__ seg_P, const int* __restrict__ cta_cnt,
                                                   int G, int64_t T, int C, int64_t n, int32_t* __restrict__ J,
                                                   double* __restrict__ PJ, int64_t* r_out) {
  __shared__ long long sh[2][8];
  const int b = blockIdx.x, tid = threadIdx.x;
  long long off = 0, tot = 0;
  for (int q = tid; q < G; q += blockDim.x) {
    const int v = cta_cnt[q];
    tot += v;
    if (q < b) off += v;
  }
  for (int o = 16; o > 0; o >>= 1) {
    off += __shfl_xor_sync(0xffffffffu, off, o);
    tot += __shfl_xor_sync(0xffffffffu, tot, o);
  }
  if ((tid & 31) == 0) {
    sh[0][tid >> 5] = off;
    sh[1][tid >> 5] = tot;
  }
  __syncthreads();
  off = 0;
  tot = 0;
  for (int wi = 0; wi < (int)(blockDim.x >> 5); ++wi) {
    off += sh[0][wi];
    tot += sh[1][wi];
  }
  if (b == 0 && tid == 0) *r_out = tot;
  int64_t c_lo, c_hi;
  cta_cols(b, G, T, C, n, &c_lo, &c_hi);
  const int cnt = cta_cnt[b];
  for (int i = tid; i < cnt; i += blockDim.x) {
    J[off + i] = seg_idx[c_lo + i];
    PJ[off + i] = seg_P[c_lo + i];
  }
}

// ---------------------------------------------------------------------------
// K5: evaluation reduce at point y (single CTA, deterministic order).
//   gp = Σ_{valid b} part_vec[b]   (b ascending)
//   g  = (y + b) − gp; ψ = ½yᵀy + bᵀy + cψ Σ P²;  res1 = ‖g‖/(1+‖b‖)
// ---------------------------------------------------------------------------
struct EvalOut {
  double psi, psimag, res1;
  double yy, by, gg;
  double s[4];      // Σ P², Σ (x−P)², Σ z², Σ ((|w|−λ1)_+)²
  double gd;        // gᵀd of the direction computed at this point (filled later)
  long long r;      // |J|
  long long pad;
};

constexpr int K5_THREADS = 1024;

__global__ void __launch_bounds__(K5_THREADS) k_eval_reduce(int64_t m, const double* __restrict__ y,
                                                            const double* __restrict__ bvec,
                                                            const double* __restrict__ part_vec,
                                                            const int* __restrict__ part_valid, int nparts,
                                                            const double* __restrict__ part_scal, int nscal,
                                                            Scal sc, double nb, int with_grad,
                                                            double* __restrict__ g_out, const int64_t* r_in,
                                                            EvalOut* out) {
  __shared__ double red[3][K5_THREADS / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double yy = 0.0, by = 0.0, gg = 0.0;
  for (int64_t k = tid; k < m; k += K5_THREADS) {
    const double yk = y[k], bk = bvec[k];
    yy += yk * yk;
    by += bk * yk;
    if (with_grad) {
      double gp = 0.0;
      int b = 0;
      for (; b + 4 <= nparts; b += 4) {  // independent loads, ordered adds
        const double v0 = (!part_valid || part_valid[b + 0]) ? part_vec[(size_t)(b + 0) * m + k] : 0.0;
        const double v1 = (!part_valid || part_valid[b + 1]) ? part_vec[(size_t)(b + 1) * m + k] : 0.0;
        const double v2 = (!part_valid || part_valid[b + 2]) ? part_vec[(size_t)(b + 2) * m + k] : 0.0;
        const double v3 = (!part_valid || part_valid[b + 3]) ? part_vec[(size_t)(b + 3) * m + k] : 0.0;
        gp += v0;
        gp += v1;
        gp += v2;
        gp += v3;
      }
      for (; b < nparts; ++b)
        if (!part_valid || part_valid[b]) gp += part_vec[(size_t)b * m + k];
      const double g = __dsub_rn(__dadd_rn(yk, bk), gp);
      g_out[k] = g;
      gg += g * g;
    }
  }
  yy = warp_allsum(yy);
  by = warp_allsum(by);
  gg = warp_allsum(gg);
  if (lane == 0) {
    red[0][warp] = yy;
    red[1][warp] = by;
    red[2][warp] = gg;
  }
  __syncthreads();
  if (tid == 0) {
    double a = 0, bb = 0, c = 0;
    for (int wi = 0; wi < K5_THREADS / 32; ++wi) {
      a += red[0][wi];
      bb += red[1][wi];
      c += red[2][wi];
    }
    double s[4] = {0, 0, 0, 0};
    for (int q = 0; q < nscal; ++q)
      for (int j = 0; j < 4; ++j) s[j] += part_scal[q * 4 + j];
    EvalOut o;
    o.yy = a;
    o.by = bb;
    o.gg = c;
    for (int j = 0; j < 4; ++j) o.s[j] = s[j];
    const double tprox = sc.cpsi * s[0];
    o.psi = 0.5 * a + bb + tprox;
    o.psimag = fabs(0.5 * a) + fabs(bb) + fabs(tprox);
    o.res1 = with_grad ? sqrt(c) / (1.0 + nb) : -1.0;
    o.gd = 0.0;
    o.r = r_in ? (long long)*r_in : -1;
    o.pad = 0;
    *out = o;
  }
}

// max over G plain-mode partials (λmax = ‖Aᵀb‖∞)
__global__ void k_max_partials(const double* part_scal, int G, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double v = 0.0;
    for (int q = 0; q < G; ++q) v = fmax(v, part_scal[q * 4]);
    *out = v;
  }
}

}  // namespace ssn
