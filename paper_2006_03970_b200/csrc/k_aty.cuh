// k_aty.cuh — the full-width pass over A and its epilogue-only twin.
//
// K1  k1_aty_fused   : w = Aᵀy over all n columns (the only O(mn) step of a Newton
//                      iteration), fused with t = x − σw, P = prox_{σp}(t) (Eq. (6),
//                      P:170-175), the active mask |t| > σλ1 (Eq. (17)),
//                      ordered compaction of (J, P_J) into per-CTA segments, block
//                      partial sums for ψ / res3 / the dual objective, and the per-CTA
//                      m-vector Σ_{i∈J} P_i a_i used by ∇ψ (Eq. (15)).
//                      Layout: one persistent CTA per SM owns a contiguous column range.
//                      A (and x) tiles stream HBM → smem through a ring of 1D bulk copies
//                      (cp.async.bulk = TMA, SASS UBLKCP) issued by one producer lane; each
//                      of 7 consumer warps owns whole tiles (tile it → warp it mod 7), so
//                      warps never wait on each other.  A warp computes 8 column dots at a
//                      time with y in registers (lane ℓ owns rows ℓ + 32t), then a
//                      transpose-reduce leaves column c's sum in lanes 4c..4c+3: the
//                      epilogue runs lane-parallel, the active flags of 8 columns become one
//                      byte of a bitmap.  Compaction happens once per CTA at the end from
//                      that bitmap (P recomputed bit-identically from the stored w).
// K1e k1e_epilogue   : the same epilogue from a stored w (or w0 + s(w1 − w0) for an
//                      Armijo backtrack, by linearity of Aᵀ), no A traffic.
// K1f k1_finalize    : concatenates the per-CTA segments in CTA order → ascending J.
// K5  k_eval_reduce  : g = y + b − Σ parts, ψ (Prop. 2), res1 (Eq. (20)).
#pragma once
#include <cooperative_groups.h>
#include "common.cuh"

namespace ssn {

constexpr int K1_NWC = 7;                     // consumer warps (7 + producer = 256 threads → 255-register cap)
constexpr int K1_THREADS = (K1_NWC + 1) * 32; // + 1 producer warp
constexpr int K1_GRP = 8;                     // columns per transpose-reduce group

struct K1Params {
  const double* A;
  int64_t m, n;
  const double* y;      // m, evaluation point
  const double* x;      // n, dense multiplier (fused mode)
  double* w_out;        // n
  uint8_t* mask;        // n/8 (+pad): active bits, one byte per 8-column group
  int32_t* seg_idx;     // n-capacity segment storage (CTA b writes from c_lo(b))
  double* seg_P;        // n
  int* cta_cnt;         // G
  double* part_scal;    // G x 4
  double* part_vec;     // G x m (fused mode; rows Σ P_i a_i)
  Scal sc;
  const Scal* scp;      // graph mode: σ-dependent scalars on the device (overrides sc)
  unsigned long long* tstamp;  // nullable: [0] ← min CTA start, [1] ← max CTA end (globaltimer ns)
  int C;                // columns per tile (multiple of 8)
  int64_t T;            // tiles
  int stages;
  int fused;            // 0: plain w = Aᵀy (+ max|w|), 1: full epilogue
  uint32_t stage_elems; // doubles per A stage buffer (≥ C*m, multiple of 16)
  uint32_t xstage_elems;// doubles per x stage buffer (≥ C, multiple of 16)
  // packed genotype storage (K1g); A == nullptr
  const uint8_t* codes; // n × cstride bytes: 2-bit codes, row k in bits 2(k%4) of byte k/4
  const double* tab;    // n × 3: decoded value of codes 0, 1, 2 for each column
  int64_t cstride;      // bytes per column (multiple of 16)
  uint32_t bfr_off;     // K1g: byte offset of the shared B-fragment table (32 k-blocks × 32 lanes × 8 B)
  // Reuse of Aᵀb (option reuse_atb, DESIGN R40; K1 and K1g): while the active set is empty (a cold
  // start's first Newton steps: x = 0, J = ∅ ⇒ g = y + b, d = −g) the trial point y + d is −b, and
  // Aᵀ(−b) = −(Aᵀb) bitwise, the product ssnal_en_create formed for λmax.  When atb != nullptr and the
  // solve's gate allowed it (the REUSE instantiation of the kernel is launched: host-driven mode, or
  // the handle's second solve graph) the launch compares y with −b bit for bit and, if equal, takes
  // w = −atb instead of streaming A: same outputs, bit for bit.  The plain instantiation carries no
  // such branch (it cost the n = 1e5 launch 5 µs of code generation: 62.9 → 68.0 µs, same-box A/B).
  const double* atb;    // n: Aᵀb kept by create (REUSE instantiation only)
  const double* bvec;   // m: b
  // REUSE instantiation: how a launch at y == −b is served.  rmode (host value, or *rmodep in graph mode):
  //   1: from atb, with the ∇ψ rows gathered from the active columns (every output of the stream);
  //   2: from atb, ψ only — no ∇ψ rows (they are worth a large part of a pass when most columns are
  //      active at −b, and Armijo usually rejects s = 1 there, after which the gradient is recomputed at
  //      the accepted step anyway); *gmiss ← 1 tells the control to redo the launch streamed if it accepts
  //      s = 1 after all;  0: stream.
  // pred (nullable): the launch runs only if *pred != 0 (the redo node of the graph); force_stream: never
  // serve from atb (the redo).  gmiss (nullable): ← 0 by a streamed launch, ← 1 by a ψ-only one.
  int rmode;
  const int* rmodep;
  const int* pred;
  int force_stream;
  int* gmiss;
};

// Reduce-scatter of 8 per-lane partial sums a[0..7] across the warp: afterwards every
// lane holds the full sum of column (lane >> 2); lanes 4c..4c+3 are bitwise identical.
SSN_DEV double reduce8(double (&a)[8], int lane) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const bool up = lane & 16;
    const double send = up ? a[j] : a[j + 4];
    const double keep = up ? a[j + 4] : a[j];
    a[j] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const bool up = lane & 8;
    const double send = up ? a[j] : a[j + 2];
    const double keep = up ? a[j + 2] : a[j];
    a[j] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  {
    const bool up = lane & 4;
    const double send = up ? a[0] : a[1];
    const double keep = up ? a[1] : a[0];
    a[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  a[0] += __shfl_xor_sync(0xffffffffu, a[0], 2);
  a[0] += __shfl_xor_sync(0xffffffffu, a[0], 1);
  return a[0];
}

// CTA end of K1 / K1g (consumer warps only; the ring is idle and holds the warps' ∇ψ partial
// rows rv[warp][0..m) when fused): fixed-order reductions of the partial scalars and rows, then
// the ordered compaction of this CTA's active columns from the bitmap (P recomputed from w).
SSN_DEV void k1_cta_end(const K1Params& p, const Scal& sc, double* ring, int* sh, int64_t c_lo, int64_t c_hi,
                        double s0, double s1, double s2, double s3, bool any_active, bool stamp = true) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m = p.m;
  double* rv = ring;                       // K1_NWC x m
  double* rs = ring + (size_t)K1_NWC * m;  // K1_NWC x 4
  int* ract = reinterpret_cast<int*>(rs + K1_NWC * 4);
  // warp partial scalars: leader lanes 0,4,...,28 in lane order (plain mode: max over lanes)
  double q4[4] = {s0, s1, s2, s3};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    double acc = 0.0;
    for (int l = 0; l < 32; l += 4) {
      const double v = __shfl_sync(0xffffffffu, q4[j], l);
      acc = p.fused ? __dadd_rn(acc, v) : fmax(acc, v);
    }
    if (!p.fused) acc = warp_allmax(q4[j]);
    q4[j] = acc;
  }
  const bool wact = __any_sync(0xffffffffu, any_active);
  if (lane == 0) {
    for (int j = 0; j < 4; ++j) rs[warp * 4 + j] = q4[j];
    ract[warp] = wact ? 1 : 0;
  }
  named_bar_sync(1, K1_NWC * 32);
  const int tid = threadIdx.x;
  const int b = blockIdx.x;
  if (tid == 0) {
    double q[4] = {rs[0], rs[1], rs[2], rs[3]};
    for (int wi = 1; wi < K1_NWC; ++wi)
      for (int j = 0; j < 4; ++j) q[j] = p.fused ? __dadd_rn(q[j], rs[wi * 4 + j]) : fmax(q[j], rs[wi * 4 + j]);
    for (int j = 0; j < 4; ++j) p.part_scal[b * 4 + j] = q[j];
  }
  // kernel-duration stamp: all consumer warps of this CTA are past their last write
  auto stamp_end = [&]() {
    if (p.tstamp && stamp) {
      named_bar_sync(1, K1_NWC * 32);
      if (tid == 0) atomicMax(p.tstamp + 1, global_ns());
    }
  };
  if (!p.fused) {
    if (tid == 0) p.cta_cnt[b] = 0;
    stamp_end();
    return;
  }
  int anyv = 0;
  for (int wi = 0; wi < K1_NWC; ++wi) anyv |= ract[wi];
  if (p.part_vec && anyv) {
    for (int64_t k = tid; k < m; k += K1_NWC * 32) {
      double v = 0.0;
      for (int wi = 0; wi < K1_NWC; ++wi)
        if (ract[wi]) v += rv[(size_t)wi * m + k];
      p.part_vec[(size_t)b * m + k] = v;
    }
  }
  if (!anyv) {
    if (tid == 0) p.cta_cnt[b] = 0;
    stamp_end();
    return;
  }
  // ordered compaction: warp wi scans bytes [bw0, bw1) of this CTA's mask range
  const int64_t byte_lo = c_lo >> 3, nbytes = (c_hi - c_lo + 7) >> 3;
  const int64_t bw0 = byte_lo + nbytes * warp / K1_NWC, bw1 = byte_lo + nbytes * (warp + 1) / K1_NWC;
  int cnt = 0;
  for (int64_t q = bw0 + lane; q < bw1; q += 32) cnt += __popc((unsigned)p.mask[q]);
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if (lane == 0) sh[warp] = cnt;
  named_bar_sync(1, K1_NWC * 32);
  int off = 0, tot = 0;
  for (int wi = 0; wi < K1_NWC; ++wi) {
    off += (wi < warp) ? sh[wi] : 0;
    tot += sh[wi];
  }
  if (tid == 0) p.cta_cnt[b] = tot;
  for (int64_t q0 = bw0; q0 < bw1; q0 += 32) {
    const int64_t q = q0 + lane;
    const unsigned byte = (q < bw1) ? (unsigned)p.mask[q] : 0u;
    const int pc = __popc(byte);
    int incl = pc;  // inclusive warp scan
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    int pos = off + incl - pc;
    unsigned bb = byte;
    while (bb) {
      const int bit = __ffs(bb) - 1;
      bb &= bb - 1;
      const int64_t i = (q << 3) + bit;
      const double w = p.w_out[i];
      const double tt = __dsub_rn(p.x[i], __dmul_rn(sc.sigma, w));
      p.seg_idx[c_lo + pos] = (int32_t)i;
      p.seg_P[c_lo + pos] = prox_en(tt, sc.thr, sc.den);
      ++pos;
    }
    off += __shfl_sync(0xffffffffu, incl, 31);
  }
  stamp_end();
}

// acc += v when (word & bit) != 0 — a predicated add, no branch (K1g's inner loop)
SSN_DEV void add_if_bit(double& acc, double v, uint32_t word, uint32_t bit) {
  asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\tand.b32 t, %2, %3;\n\tsetp.ne.u32 p, t, 0;\n\t@p add.f64 %0, %0, %1;\n\t}"
      : "+d"(acc)
      : "d"(v), "r"(word), "r"(bit));
}
// x = v when (word & bit) != 0 — a predicated move
SSN_DEV void sel_if_bit(double& x, double v, uint32_t word, uint32_t bit) {
  asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\tand.b32 t, %2, %3;\n\tsetp.ne.u32 p, t, 0;\n\t@p mov.f64 %0, %1;\n\t}"
      : "+d"(x)
      : "d"(v), "r"(word), "r"(bit));
}

// K1 served from the kept product Aᵀb (K1Params::atb): w_i = −atb_i instead of the dot product, the
// same epilogue on the same (warp, lane, order) assignment of columns as the streaming kernel, the
// ∇ψ partial rows from the active columns read straight from global memory — every output (w, mask,
// segments, partial scalars and rows) is bitwise what the streaming launch at y = −b writes.  No ring,
// no producer; kD groups of (w, x) loads in flight per warp.  Not stamped (it is not a pass over A).
// GENO: packed genotype storage (K1g's layout of the ∇ψ partial rows: lane ℓ owns code words ℓ + 32t,
// 16 rows each; MR = TW words per lane).
template <int MR, bool GENO = false>
SSN_DEV void k1_cached(const K1Params& p, double* ring, int* sh, int64_t c_lo, int64_t c_hi, bool psi_only) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == K1_NWC) return;
  constexpr int kD = 8;
  const int C = p.C;
  const int64_t m = p.m;
  const int64_t ntiles = (c_hi - c_lo + C - 1) / C;
  const int gpt = C / K1_GRP;  // groups per tile
  constexpr int NG = GENO ? 16 * MR : MR;
  double gacc[NG];
#pragma unroll
  for (int t = 0; t < NG; ++t) gacc[t] = 0.0;
  const int nwords = (int)(p.cstride >> 2);
  const Scal sc = p.scp ? *p.scp : p.sc;
  const bool leader = (lane & 3) == 0;
  const int gcol = lane >> 2;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  bool any_active = false;
  const int ntw = ntiles > warp ? (int)((ntiles - warp + K1_NWC - 1) / K1_NWC) : 0;  // this warp's tiles
  int tk = 0, tg = 0;  // next group: tile warp + K1_NWC·tk of this CTA, group tg of it
  while (tk < ntw) {
    double wv[kD], xv[kD];
    int64_t cc[kD];   // global column of this lane in group u, −1: not a column
    int64_t gb[kD];   // first global column of group u, −1: the group does not exist
    // all loads of the batch issue back to back (clamped addresses, no branch, no use before the batch is out)
#pragma unroll
    for (int u = 0; u < kD; ++u) {
      const bool tile_ok = tk < ntw;
      const int64_t c0 = c_lo + (int64_t)(warp + K1_NWC * (tile_ok ? tk : 0)) * C;
      const int nc = (int)((c_hi - c0) < C ? (c_hi - c0) : C);
      const bool grp = tile_ok && tg * K1_GRP < nc;
      const bool col = grp && tg * K1_GRP + gcol < nc;
      gb[u] = grp ? c0 + (int64_t)tg * K1_GRP : -1;
      cc[u] = col ? gb[u] + gcol : -1;
      const int64_t ca = col ? cc[u] : c_lo;
      wv[u] = __ldg(p.atb + ca);
      xv[u] = p.fused ? __ldg(p.x + ca) : 0.0;
      if (++tg == gpt) {
        tg = 0;
        ++tk;
      }
    }
#pragma unroll
    for (int u = 0; u < kD; ++u) {
      if (gb[u] < 0) continue;  // warp-uniform
      const bool valid = cc[u] >= 0;
      const double w = -wv[u];  // Aᵀ(−b) = −(Aᵀb) bitwise
      if (p.fused) {
        bool act = false;
        double P = 0.0;
        if (valid) {
          const double xi = xv[u];
          const double tt = __dsub_rn(xi, __dmul_rn(sc.sigma, w));
          act = fabs(tt) > sc.thr;
          const double e = __dsub_rn(fabs(w), sc.l1);
          if (xi == 0.0 && !act) {
            if (leader) {
              s2 = __dadd_rn(s2, __dmul_rn(w, w));
              if (e > 0.0) s3 = __dadd_rn(s3, __dmul_rn(e, e));
            }
          } else {
            P = prox_en(tt, sc.thr, sc.den);
            const double dx = __dsub_rn(xi, P);
            const double z = __dsub_rn(__ddiv_rn(dx, sc.sigma), w);
            if (leader) {
              s0 = __dadd_rn(s0, __dmul_rn(P, P));
              s1 = __dadd_rn(s1, __dmul_rn(dx, dx));
              s2 = __dadd_rn(s2, __dmul_rn(z, z));
              if (e > 0.0) s3 = __dadd_rn(s3, __dmul_rn(e, e));
            }
          }
          if (leader) p.w_out[cc[u]] = w;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, act && leader);
        unsigned m8 = 0;
#pragma unroll
        for (int q = 0; q < K1_GRP; ++q) m8 |= ((bal >> (4 * q)) & 1u) << q;
        if (lane == 0) p.mask[gb[u] >> 3] = (uint8_t)m8;
        if (m8) any_active = true;
        if (m8 && !psi_only) {
          unsigned mm = m8;
          while (mm) {
            const int q = __ffs(mm) - 1;
            mm &= mm - 1;
            const double Pq = __shfl_sync(0xffffffffu, P, 4 * q);
            if constexpr (GENO) {
              const int64_t cq = gb[u] + q;
              const double v0 = __ldg(p.tab + 3 * cq), v1 = __ldg(p.tab + 3 * cq + 1), v2 = __ldg(p.tab + 3 * cq + 2);
              const uint32_t* wcol = reinterpret_cast<const uint32_t*>(p.codes + cq * p.cstride);
#pragma unroll
              for (int t = 0; t < MR; ++t) {
                const int wi = lane + 32 * t;
                const uint32_t word = (wi < nwords) ? __ldg(wcol + wi) : 0u;
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                  double v = v0;
                  sel_if_bit(v, v1, word, 1u << (2 * e));
                  sel_if_bit(v, v2, word, 2u << (2 * e));
                  gacc[16 * t + e] = fma(Pq, v, gacc[16 * t + e]);
                }
              }
            } else {
              const double* colq = p.A + (gb[u] + q) * m;
#pragma unroll
              for (int t = 0; t < MR; ++t) {
                const int64_t row = lane + 32 * t;
                if (row < m) gacc[t] = fma(Pq, __ldg(colq + row), gacc[t]);
              }
            }
          }
        }
      } else {
        if (valid) {
          s0 = fmax(s0, fabs(w));
          if (leader) p.w_out[cc[u]] = w;
        }
      }
    }
  }
  named_bar_sync(1, K1_NWC * 32);
  if (p.fused && p.part_vec) {
    if constexpr (GENO) {
#pragma unroll
      for (int t = 0; t < MR; ++t)
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int64_t row = 16 * (lane + 32 * t) + e;
          if (row < m) ring[(size_t)warp * m + row] = gacc[16 * t + e];
        }
    } else {
#pragma unroll
      for (int t = 0; t < MR; ++t) {
        const int64_t row = lane + 32 * t;
        if (row < m) ring[(size_t)warp * m + row] = gacc[t];
      }
    }
  }
  // ψ-only: nothing reads this trial's active set (a rejected trial is re-thresholded by the backtrack, an
  // accepted one is redone streamed): no compaction, no ∇ψ rows — the CTA reports an empty segment
  k1_cta_end(p, sc, ring, sh, c_lo, c_hi, s0, s1, s2, s3, any_active && !psi_only, false);
}

template <int MR, bool REUSE = false>
__global__ void __launch_bounds__(K1_THREADS, 1) k1_aty_fused(const K1Params p) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = p.stages, C = p.C;
  const int64_t m = p.m;
  double* ring = reinterpret_cast<double*>(smem);
  double* xring = ring + (size_t)S * p.stage_elems;
  uint64_t* full = reinterpret_cast<uint64_t*>(xring + (size_t)S * p.xstage_elems);
  uint64_t* empty = full + S;
  int* sh = reinterpret_cast<int*>(empty + S);  // small scratch (16 ints)
  volatile int* slot_seq = sh + 16;              // S ints: tile last issued into each slot

  int64_t c_lo, c_hi;
  cta_cols(blockIdx.x, gridDim.x, p.T, C, p.n, &c_lo, &c_hi);
  const int64_t ntiles = (c_hi - c_lo + C - 1) / C;
  if constexpr (REUSE) {  // R40: y == −b ⇒ w = −Aᵀb kept by create
    if (p.pred && *p.pred == 0) return;
    const int mode = p.force_stream ? 0 : (p.rmodep ? *p.rmodep : p.rmode);
    bool eq = mode != 0;
    if (eq)
      for (int64_t row = threadIdx.x; row < m; row += K1_THREADS)
        eq = eq && (__double_as_longlong(p.y[row]) == __double_as_longlong(-p.bvec[row]));
    const bool cached = __syncthreads_and(eq);
    if (p.gmiss && blockIdx.x == 0 && threadIdx.x == 0) *p.gmiss = (cached && mode == 2) ? 1 : 0;
    if (cached) {
      k1_cached<MR>(p, ring, sh, c_lo, c_hi, mode == 2);
      return;
    }
  }

  if (threadIdx.x == 0) {
    if (p.tstamp) atomicMin(p.tstamp, global_ns());
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      slot_seq[s] = -1;
    }
    fence_mbar_init();
  }
  __syncthreads();

  // Slot s carries tiles s, s+S, s+2S, ... consumed by different warps.  A consumer must not
  // try_wait on full[s] before its own tile was issued: the parity of a phase two steps ahead
  // aliases the current one.  The producer publishes the issued tile number in slot_seq[s].
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
        slot_seq[s] = (int)it;
      }
    }
    return;
  }

  // ---------------- consumer warps: warp w owns tiles it ≡ w (mod K1_NWC) ----------------
  double yr[MR], gacc[MR];
#pragma unroll
  for (int t = 0; t < MR; ++t) {
    const int64_t row = lane + 32 * t;
    yr[t] = row < m ? p.y[row] : 0.0;
    gacc[t] = 0.0;
  }
  const Scal sc = p.scp ? *p.scp : p.sc;
  const bool leader = (lane & 3) == 0;
  const int gcol = lane >> 2;  // column of the 8-group this lane ends up holding
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;  // per leader lane, its columns in order
  bool any_active = false;

  for (int64_t it = warp; it < ntiles; it += K1_NWC) {
    const int s = (int)(it % S);
    if (lane == 0)
      while (slot_seq[s] != (int)it) __nanosleep(32);
    __syncwarp();
    mbar_wait(&full[s], (uint32_t)((it / S) & 1));
    const int64_t c0 = c_lo + it * C;
    const int nc = (int)((c_hi - c0) < C ? (c_hi - c0) : C);
    const double* Ts = ring + (size_t)s * p.stage_elems;
    const double* Xs = xring + (size_t)s * p.xstage_elems;
    for (int g = 0; g * K1_GRP < nc; ++g) {
      const double* base = Ts + (size_t)g * K1_GRP * m;
      double a[K1_GRP];
#pragma unroll
      for (int c = 0; c < K1_GRP; ++c) a[c] = 0.0;
#pragma unroll
      for (int t = 0; t < MR; ++t) {
        const int64_t row = lane + 32 * t;
        if (row < m) {
          const double yv = yr[t];
#pragma unroll
          for (int c = 0; c < K1_GRP; ++c) a[c] = fma(yv, base[(size_t)c * m + row], a[c]);
        }
      }
      const double w = reduce8(a, lane);
      const int c = g * K1_GRP + gcol;
      const bool valid = c < nc;
      if (p.fused) {
        bool act = false;
        double P = 0.0;
        if (valid) {
          const double xi = Xs[c];
          const double tt = __dsub_rn(xi, __dmul_rn(sc.sigma, w));
          act = fabs(tt) > sc.thr;
          const double e = __dsub_rn(fabs(w), sc.l1);
          if (xi == 0.0 && !act) {  // P = 0, x − P = 0, z = −w (exact shortcut of the line below)
            if (leader) {
              s2 = __dadd_rn(s2, __dmul_rn(w, w));
              if (e > 0.0) s3 = __dadd_rn(s3, __dmul_rn(e, e));
            }
          } else {
            P = prox_en(tt, sc.thr, sc.den);
            const double dx = __dsub_rn(xi, P);
            const double z = __dsub_rn(__ddiv_rn(dx, sc.sigma), w);
            if (leader) {
              s0 = __dadd_rn(s0, __dmul_rn(P, P));
              s1 = __dadd_rn(s1, __dmul_rn(dx, dx));
              s2 = __dadd_rn(s2, __dmul_rn(z, z));
              if (e > 0.0) s3 = __dadd_rn(s3, __dmul_rn(e, e));
            }
          }
          if (leader) p.w_out[c0 + c] = w;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, act && leader);
        unsigned m8 = 0;
#pragma unroll
        for (int q = 0; q < K1_GRP; ++q) m8 |= ((bal >> (4 * q)) & 1u) << q;
        if (lane == 0) p.mask[(c0 >> 3) + g] = (uint8_t)m8;
        if (m8) {
          any_active = true;
          unsigned mm = m8;
          while (mm) {
            const int q = __ffs(mm) - 1;
            mm &= mm - 1;
            const double Pq = __shfl_sync(0xffffffffu, P, 4 * q);
            const double* colq = base + (size_t)q * m;
#pragma unroll
            for (int t = 0; t < MR; ++t) {
              const int64_t row = lane + 32 * t;
              if (row < m) gacc[t] = fma(Pq, colq[row], gacc[t]);
            }
          }
        }
      } else {
        if (valid) {
          s0 = fmax(s0, fabs(w));
          if (leader) p.w_out[c0 + c] = w;
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // ---------------- CTA epilogue: fixed-order reductions, then ordered compaction ----------------
  named_bar_sync(1, K1_NWC * 32);  // ring idle; this CTA's w / mask writes are visible CTA-wide
  if (p.fused && p.part_vec) {
#pragma unroll
    for (int t = 0; t < MR; ++t) {
      const int64_t row = lane + 32 * t;
      if (row < m) ring[(size_t)warp * m + row] = gacc[t];
    }
  }
  k1_cta_end(p, sc, ring, sh, c_lo, c_hi, s0, s1, s2, s3, any_active);
}

// ---------------------------------------------------------------------------
// K1g: K1 over packed 2-bit genotype codes.  Column j is cstride bytes of
// codes g ∈ {0,1,2} and a 3-entry table v_j[g] (the standardised value, bit-exact with the
// fp64 design); a_kj = v_j[g_kj].  The A tile of a stage is C × cstride bytes of codes plus
// C × 3 table doubles, streamed by the same 1D bulk-copy ring (32× fewer bytes than fp64).
// Lane ℓ owns 32-bit words ℓ + 32t of every column (rows 16(ℓ + 32t) + 0..15, y in
// registers).  Since a_kj takes three values per column, a_jᵀy = v0 ΣY + (v1−v0) S1 + (v2−v0) S2
// with the bucket sums S_g = Σ_{k: g_kj = g} y_k: per element two bit-tested predicated adds.
// The 8-column transpose-reduce, the epilogue and the CTA end are K1's.
// ---------------------------------------------------------------------------
template <int TW, bool REUSE = false>
__global__ void __launch_bounds__(K1_THREADS, 1) k1g_aty_fused(const K1Params p) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = p.stages, C = p.C;
  const int64_t m = p.m, cs = p.cstride;
  const int nwords = (int)(cs >> 2);
  double* ring = reinterpret_cast<double*>(smem);  // per stage: codes (cs·C bytes) then table (3C doubles)
  double* xring = ring + (size_t)S * p.stage_elems;
  uint64_t* full = reinterpret_cast<uint64_t*>(xring + (size_t)S * p.xstage_elems);
  uint64_t* empty = full + S;
  int* sh = reinterpret_cast<int*>(empty + S);
  volatile int* slot_seq = sh + 16;
  const uint32_t code_elems = (uint32_t)((cs * C + 7) / 8);  // doubles occupied by a stage's codes

  int64_t c_lo, c_hi;
  cta_cols(blockIdx.x, gridDim.x, p.T, C, p.n, &c_lo, &c_hi);
  const int64_t ntiles = (c_hi - c_lo + C - 1) / C;
  if constexpr (REUSE) {  // R40: y == −b ⇒ w = −Aᵀb kept by create (Aᵀ(−y) = −Aᵀy bitwise here too: rint is odd)
    if (p.pred && *p.pred == 0) return;
    const int mode = p.force_stream ? 0 : (p.rmodep ? *p.rmodep : p.rmode);
    bool eq = mode != 0;
    if (eq)
      for (int64_t row = threadIdx.x; row < m; row += K1_THREADS)
        eq = eq && (__double_as_longlong(p.y[row]) == __double_as_longlong(-p.bvec[row]));
    const bool cached = __syncthreads_and(eq);
    if (p.gmiss && blockIdx.x == 0 && threadIdx.x == 0) *p.gmiss = (cached && mode == 2) ? 1 : 0;
    if (cached) {
      k1_cached<TW, true>(p, ring, sh, c_lo, c_hi, mode == 2);
      return;
    }
  }
  if (threadIdx.x == 0) {
    if (p.tstamp) atomicMin(p.tstamp, global_ns());
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      slot_seq[s] = -1;
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
        double* dst = ring + (size_t)s * p.stage_elems;
        double* dT = dst + code_elems;
        double* dX = xring + (size_t)s * p.xstage_elems;
        const uint32_t bytesC = (uint32_t)(nc * cs);  // multiple of 16
        const uint32_t bytesT = (uint32_t)nc * 24u, t16 = bytesT & ~15u;
        if (t16 != bytesT) dT[3 * nc - 1] = __ldg(p.tab + (c0 + nc) * 3 - 1);  // 8-B tail
        uint32_t x16 = 0;
        if (p.fused) {
          const uint32_t bytesX = (uint32_t)nc * 8u;
          x16 = bytesX & ~15u;
          if (x16 != bytesX) dX[nc - 1] = __ldg(p.x + c0 + nc - 1);
        }
        fence_proxy_async();
        mbar_arrive_expect_tx(&full[s], bytesC + t16 + x16);
        bulk_g2s(dst, p.codes + c0 * cs, bytesC, &full[s]);
        if (t16) bulk_g2s(dT, p.tab + c0 * 3, t16, &full[s]);
        if (x16) bulk_g2s(dX, p.x + c0, x16, &full[s]);
        slot_seq[s] = (int)it;
      }
    }
    return;
  }

  // ---------------- consumer warps ----------------
  // a_jᵀy = v0 ΣY + (v1 − v0) S1 + (v2 − v0) S2 with the bucket sums S_g = Σ_{k: g_kj = g} y_k.  The
  // bucket sums are exact integer dot products on the INT8 tensor cores (mma.sync m16n8k32 u8,
  // SASS IMMA): y is rounded once to 64-bit fixed point Y = rint(y·2^e) (2^e the largest power of two
  // with m·max|y|·2^e < 2^62, so every partial sum fits), split into 8 byte limbs (the B operand:
  // 32 rows × 8 limbs, kept in registers for the whole launch), and each column's code bytes expand
  // to the 0/1 bit planes [g = 1], [g = 2] (the A operand: 16 columns × 32 rows; code 3 is rejected
  // at create, so g = 1 ⇔ bit 0, g = 2 ⇔ bit 1).  The int32 accumulators per limb are exact
  // (≤ 1024 · 255); Σ_l C_l 2^{8l} mod 2^64 is the exact two's-complement S·2^e, converted to fp64
  // once.  Rounding y costs ≤ m·2^{-e-1} ≈ m²·max|y|·2^{-63} per bucket sum, ~1e-13 of the R21 bound
  // (DESIGN.md §5).  Thread (g = lane/4, t = lane%4) of the warp's 16-column group: A rows (columns)
  // g and g + 8, k = 4t … 4t + 3 and 16 + 4t …; B limb g of the same k; C columns (limbs) 2t, 2t + 1.
  const int gq = lane >> 2, tq = lane & 3;
  const int nkb = (int)((m + 31) / 32);
  double ysum = 0.0, ymax = 0.0;  // Σ y (fixed lane then butterfly order), max |y|
  for (int64_t row = lane; row < m; row += 32) {
    const double yv = p.y[row];
    ysum += yv;
    ymax = fmax(ymax, fabs(yv));
  }
  ysum = warp_allsum(ysum);
  ymax = warp_allmax(ymax);
  int ex = 0;
  if (ymax > 0.0) {
    int e2;
    frexp(ymax * (double)m, &e2);  // m·max|y| < 2^e2
    ex = 62 - e2;
  }
  const double unscale = ldexp(1.0, -ex);
  // B fragments (limb gq of Y at rows 32kb + 4tq + i and 32kb + 16 + 4tq + i), identical for every
  // warp: built once per CTA into shared memory, read per k-block (conflict-free: entry kb·32 + lane)
  uint2* bsm = reinterpret_cast<uint2*>(smem + p.bfr_off);
  for (int kb = warp; kb < 32; kb += K1_NWC) {
    uint32_t v[2] = {0u, 0u};
    if (kb < nkb) {
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int64_t row = 32 * kb + 16 * h + 4 * tq + i;
          const long long Y = row < m ? __double2ll_rn(ldexp(p.y[row], ex)) : 0ll;
          v[h] |= (uint32_t)(((unsigned long long)Y >> (8 * gq)) & 0xFFull) << (8 * i);
        }
    }
    bsm[kb * 32 + lane] = make_uint2(v[0], v[1]);
  }
  named_bar_sync(1, K1_NWC * 32);
  double gacc[TW][16];
#pragma unroll
  for (int t = 0; t < TW; ++t)
#pragma unroll
    for (int q = 0; q < 16; ++q) gacc[t][q] = 0.0;
  const Scal sc = p.scp ? *p.scp : p.sc;
  const bool leader = (lane & 3) == 0;
  const int gcol = lane >> 2;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  bool any_active = false;

  // code byte → 4 bytes of the bit plane (bit `sh` of each 2-bit code): the set bits 0, 2, 4, 6 of
  // (x >> sh) & 0x55 move to bits 0, 8, 16, 24 by one multiply (carries land on odd bit positions)
  auto plane = [](uint32_t x, int sh) { return (((x >> sh) & 0x55u) * 0x41041u) & 0x01010101u; };
  auto imma = [](int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  };
  // Σ_l C_l 2^{8l} over the quad's limbs (mod 2^64), for this thread's two C rows
  auto limbs = [&](const int (&c)[4], unsigned long long& ra, unsigned long long& rb) {
    ra = ((unsigned long long)(long long)c[0] << (16 * tq)) + ((unsigned long long)(long long)c[1] << (16 * tq + 8));
    rb = ((unsigned long long)(long long)c[2] << (16 * tq)) + ((unsigned long long)(long long)c[3] << (16 * tq + 8));
#pragma unroll
    for (int o = 1; o < 4; o <<= 1) {
      ra += __shfl_xor_sync(0xffffffffu, ra, o);
      rb += __shfl_xor_sync(0xffffffffu, rb, o);
    }
  };

  for (int64_t it = warp; it < ntiles; it += K1_NWC) {
    const int s = (int)(it % S);
    if (lane == 0)
      while (slot_seq[s] != (int)it) __nanosleep(32);
    __syncwarp();
    mbar_wait(&full[s], (uint32_t)((it / S) & 1));
    const int64_t c0 = c_lo + it * C;
    const int nc = (int)((c_hi - c0) < C ? (c_hi - c0) : C);
    const unsigned char* Cs = reinterpret_cast<const unsigned char*>(ring + (size_t)s * p.stage_elems);
    const double* Ts = ring + (size_t)s * p.stage_elems + code_elems;
    const double* Xs = xring + (size_t)s * p.xstage_elems;

    // epilogue of the 8-column group g (lanes 4c … 4c + 3 hold column g·8 + c's value w)
    auto epi8 = [&](int g, double w) {
      const int c = g * K1_GRP + gcol;
      const bool valid = c < nc;
      if (p.fused) {
        bool act = false;
        double P = 0.0;
        if (valid) {
          const double xi = Xs[c];
          const double tt = __dsub_rn(xi, __dmul_rn(sc.sigma, w));
          act = fabs(tt) > sc.thr;
          const double e = __dsub_rn(fabs(w), sc.l1);
          if (xi == 0.0 && !act) {
            if (leader) {
              s2 = __dadd_rn(s2, __dmul_rn(w, w));
              if (e > 0.0) s3 = __dadd_rn(s3, __dmul_rn(e, e));
            }
          } else {
            P = prox_en(tt, sc.thr, sc.den);
            const double dx = __dsub_rn(xi, P);
            const double z = __dsub_rn(__ddiv_rn(dx, sc.sigma), w);
            if (leader) {
              s0 = __dadd_rn(s0, __dmul_rn(P, P));
              s1 = __dadd_rn(s1, __dmul_rn(dx, dx));
              s2 = __dadd_rn(s2, __dmul_rn(z, z));
              if (e > 0.0) s3 = __dadd_rn(s3, __dmul_rn(e, e));
            }
          }
          if (leader) p.w_out[c0 + c] = w;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, act && leader);
        unsigned m8 = 0;
#pragma unroll
        for (int q = 0; q < K1_GRP; ++q) m8 |= ((bal >> (4 * q)) & 1u) << q;
        if (lane == 0) p.mask[(c0 >> 3) + g] = (uint8_t)m8;
        if (m8) {
          any_active = true;
          unsigned mm = m8;
          while (mm) {
            const int q8 = __ffs(mm) - 1;
            mm &= mm - 1;
            const double Pq = __shfl_sync(0xffffffffu, P, 4 * q8);
            const int cq = g * K1_GRP + q8;
            const double v0 = Ts[3 * cq], v1 = Ts[3 * cq + 1], v2 = Ts[3 * cq + 2];
            const uint32_t* wcol = reinterpret_cast<const uint32_t*>(Cs + (size_t)cq * cs);
#pragma unroll
            for (int t = 0; t < TW; ++t) {
              const int wi = lane + 32 * t;
              const uint32_t word = (wi < nwords) ? wcol[wi] : 0u;
#pragma unroll
              for (int q = 0; q < 16; ++q) {
                double v = v0;
                sel_if_bit(v, v1, word, 1u << (2 * q));
                sel_if_bit(v, v2, word, 2u << (2 * q));
                gacc[t][q] = fma(Pq, v, gacc[t][q]);
              }
            }
          }
        }
      } else {
        if (valid) {
          s0 = fmax(s0, fabs(w));
          if (leader) p.w_out[c0 + c] = w;
        }
      }
    };

    // two 16-column groups per iteration (independent chains: the loop is latency-, not pipe-bound)
    for (int g32 = 0; g32 * 32 < nc; ++g32) {
      int cA[2], cB[2];
      bool vA[2], vB[2];
      const unsigned char* pA[2];
      const unsigned char* pB[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        cA[u] = g32 * 32 + 16 * u + gq;  // this thread's A rows (columns) of group u
        cB[u] = cA[u] + 8;
        vA[u] = cA[u] < nc;
        vB[u] = cB[u] < nc;
        pA[u] = Cs + (size_t)(vA[u] ? cA[u] : 0) * cs;
        pB[u] = Cs + (size_t)(vB[u] ? cB[u] : 0) * cs;
      }
      int acc1[2][4], acc2[2][4];  // [group][C fragment], planes [g = 1], [g = 2]
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc1[u][e] = acc2[u][e] = 0;
#pragma unroll
      for (int kb = 0; kb < 32; ++kb) {
        if (kb < nkb) {
          const uint2 bb = bsm[kb * 32 + lane];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const uint2 wa = vA[u] ? *reinterpret_cast<const uint2*>(pA[u] + 8 * kb) : make_uint2(0u, 0u);
            const uint2 wb = vB[u] ? *reinterpret_cast<const uint2*>(pB[u] + 8 * kb) : make_uint2(0u, 0u);
            const uint32_t xa0 = (wa.x >> (8 * tq)) & 0xFFu, xa1 = (wa.y >> (8 * tq)) & 0xFFu;
            const uint32_t xb0 = (wb.x >> (8 * tq)) & 0xFFu, xb1 = (wb.y >> (8 * tq)) & 0xFFu;
            imma(acc1[u], plane(xa0, 0), plane(xb0, 0), plane(xa1, 0), plane(xb1, 0), bb.x, bb.y);
            imma(acc2[u], plane(xa0, 1), plane(xb0, 1), plane(xa1, 1), plane(xb1, 1), bb.x, bb.y);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (g32 * 32 + 16 * u >= nc) break;
        unsigned long long s1a, s1b, s2a, s2b;
        limbs(acc1[u], s1a, s1b);
        limbs(acc2[u], s2a, s2b);
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          const int cc = half ? cB[u] : cA[u];
          const bool cv = cc < nc;
          const double S1 = (double)(long long)(half ? s1b : s1a) * unscale;
          const double S2 = (double)(long long)(half ? s2b : s2a) * unscale;
          const double v0 = cv ? Ts[3 * cc] : 0.0, v1 = cv ? Ts[3 * cc + 1] : 0.0, v2 = cv ? Ts[3 * cc + 2] : 0.0;
          const double w = fma(v2 - v0, S2, fma(v1 - v0, S1, v0 * ysum));
          const int g8 = g32 * 4 + 2 * u + half;
          if (g8 < (nc + K1_GRP - 1) / K1_GRP) epi8(g8, w);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  named_bar_sync(1, K1_NWC * 32);  // ring idle
  if (p.fused && p.part_vec) {
#pragma unroll
    for (int t = 0; t < TW; ++t)
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int64_t row = 16 * (lane + 32 * t) + q;
        if (row < m) ring[(size_t)warp * m + row] = gacc[t][q];
      }
  }
  k1_cta_end(p, sc, ring, sh, c_lo, c_hi, s0, s1, s2, s3, any_active);
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
  const Scal* scp;   // graph mode: device scalars (overrides sc)
  const double* sp;  // graph mode: device step length (overrides s)
  int C;
  int64_t T;
};

// Each iteration covers K1E_U · K1E_THREADS consecutive columns (element u of thread t is column
// base + u·K1E_THREADS + t: coalesced per u), with all loads issued before any use so that
// 3 · K1E_U loads per thread are in flight (an HBM stream needs ~40 KB in flight per SM; one load
// per thread and two barriers per 512 columns left the round-1 version latency-bound at ~11% of its
// roofline).  The compaction stays ordered: warp counts per u, one barrier, prefix over (u, warp).
constexpr int K1E_U = 8;
__global__ void __launch_bounds__(K1E_THREADS) k1e_epilogue(const K1eParams p) {
  constexpr int NW = K1E_THREADS / 32;
  constexpr int NE = K1E_U * NW;  // (u, warp) count entries per iteration, u-major = column order
  static_assert(NE % 32 == 0, "scan layout");
  __shared__ int wcnt[2][NE];     // double-buffered by iteration parity (no end-of-iteration barrier)
  __shared__ int offs[2][NE + 1]; // exclusive prefix; [NE] = iteration total
  __shared__ double red[NW][4];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int64_t c_lo, c_hi;
  cta_cols(blockIdx.x, gridDim.x, p.T, p.C, p.n, &c_lo, &c_hi);
  const Scal sc = p.scp ? *p.scp : p.sc;
  const double step = p.sp ? *p.sp : p.s;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int64_t cnt = 0;
  int par = 0;
  const unsigned lt = lanemask_lt();
  for (int64_t base = c_lo; base < c_hi; base += (int64_t)K1E_U * K1E_THREADS, par ^= 1) {
    double wv[K1E_U], xv[K1E_U], w1v[K1E_U];
#pragma unroll
    for (int u = 0; u < K1E_U; ++u) {
      const int64_t i = base + (int64_t)u * K1E_THREADS + tid;
      const bool in = i < c_hi;
      wv[u] = in ? __ldg(p.w0 + i) : 0.0;
      xv[u] = in ? __ldg(p.x + i) : 0.0;
      w1v[u] = (in && p.w1) ? __ldg(p.w1 + i) : 0.0;
    }
    unsigned bal[K1E_U];
    double Pv[K1E_U];
#pragma unroll
    for (int u = 0; u < K1E_U; ++u) {
      const int64_t i = base + (int64_t)u * K1E_THREADS + tid;
      int act = 0;
      double P = 0.0;
      if (i < c_hi) {
        double w = wv[u];
        if (p.w1) w = __dadd_rn(w, __dmul_rn(step, __dsub_rn(w1v[u], w)));
        if (p.w_out) p.w_out[i] = w;
        const double xi = xv[u];
        const double tt = __dsub_rn(xi, __dmul_rn(sc.sigma, w));
        act = fabs(tt) > sc.thr;
        const double e = __dsub_rn(fabs(w), sc.l1);
        if (xi == 0.0 && !act) {  // P = 0, x − P = 0, z = 0/σ − w = −w exactly: no division (as in K1)
          s2 = __dadd_rn(s2, __dmul_rn(w, w));
        } else {
          P = prox_en(tt, sc.thr, sc.den);
          const double dx = __dsub_rn(xi, P);
          const double z = __dsub_rn(__ddiv_rn(dx, sc.sigma), w);
          s0 = __dadd_rn(s0, __dmul_rn(P, P));
          s1 = __dadd_rn(s1, __dmul_rn(dx, dx));
          s2 = __dadd_rn(s2, __dmul_rn(z, z));
        }
        if (e > 0.0) s3 = __dadd_rn(s3, __dmul_rn(e, e));
      }
      Pv[u] = P;
      bal[u] = __ballot_sync(0xffffffffu, act);
      if (lane == 0) wcnt[par][u * NW + warp] = __popc(bal[u]);
    }
    __syncthreads();
    if (warp == 0) {  // exclusive scan of the NE counts in column order: lane owns NE/32 consecutive entries
      constexpr int PL = NE / 32;
      int v[PL], sum = 0;
#pragma unroll
      for (int j = 0; j < PL; ++j) {
        v[j] = wcnt[par][lane * PL + j];
        sum += v[j];
      }
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      int run = incl - sum;
#pragma unroll
      for (int j = 0; j < PL; ++j) {
        offs[par][lane * PL + j] = run;
        run += v[j];
      }
      if (lane == 31) offs[par][NE] = incl;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < K1E_U; ++u)
      if (bal[u] & (1u << lane)) {
        const int64_t pos = cnt + offs[par][u * NW + warp] + __popc(bal[u] & lt);
        p.seg_idx[c_lo + pos] = (int32_t)(base + (int64_t)u * K1E_THREADS + tid);
        p.seg_P[c_lo + pos] = Pv[u];
      }
    cnt += offs[par][NE];
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
                                                   double* __restrict__ PJ, int64_t* r_out, const int* pred = nullptr) {
  if (pred && *pred == 0) return;
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
  double gd;        // gᵀd of the direction that produced this point (copied from gd_src)
  long long r;      // |J|
  long long info;   // Cholesky status of that direction (copied from info_src)
  unsigned long long seq;  // written last (mapped host copy: the host spins on it)
  unsigned long long pad;
};

constexpr int K5_THREADS = 256;  // 8 warps; CTA c owns rows [32c, 32c + 32)

// Multi-CTA, deterministic.  Clusters of kEvalCS CTAs per 32-row block rb: with the gradient,
// CTA q of the cluster sums the partial rows b ∈ [q·np/8, (q+1)·np/8) (warp w a contiguous
// eighth of that, ascending b) for the block's 32 rows; the warp sums are added in warp order
// and rank 0 adds the cluster's CTA sums in rank order through DSMEM.  Rank 0 then forms g and
// the block's scalar partials; the last row block (ticket counter) adds them in block order,
// adds the per-CTA scalar partials of K1/K1e in CTA order and writes EvalOut.
constexpr int kEvalCS = 8;
// The evaluation as a device function: true on the one thread that finishes (after *out is
// written), so control epilogues can follow in the same launch (k_ctl.cuh).
SSN_DEV bool eval_body(int64_t m, const double* __restrict__ y,
                                                            const double* __restrict__ bvec,
                                                            const double* __restrict__ part_vec,
                                                            const int* __restrict__ part_valid, int nparts,
                                                            const double* __restrict__ part_scal, int nscal,
                                                            Scal sc, double nb, int with_grad,
                                                            double* __restrict__ g_out, const int64_t* r_in,
                                                            EvalOut* out, double* blk, unsigned* ticket,
                                                            const double* gd_src, const int* info_src,
                                                            EvalOut* host_out, unsigned long long seq,
                                                            const Scal* scp, const int* pred, const double* nbp) {

  __shared__ double red[8][33];
  __shared__ bool last;
  if (pred && *pred == 0) return false;  // graph mode: predicated off (uniform over the grid)
  if (scp) sc = *scp;
  if (nbp) nb = *nbp;  // graph mode: ‖b‖ from the control block (the graph may predate it)
  namespace cg = cooperative_groups;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cs = (int)(blockIdx.x % kEvalCS), rb = (int)(blockIdx.x / kEvalCS), nrb = (int)(gridDim.x / kEvalCS);
  const int64_t k = (int64_t)rb * 32 + lane;
  __shared__ double gsum[32];
  double yk = 0.0, bk = 0.0;  // prefetched for the row-block sums below
  if (cs == 0 && warp == 0 && k < m) {
    yk = y[k];
    bk = bvec[k];
  }
  if (with_grad) {
    const int q0 = (int)((int64_t)nparts * cs / kEvalCS), q1 = (int)((int64_t)nparts * (cs + 1) / kEvalCS);
    const int b0 = q0 + (int)((int64_t)(q1 - q0) * warp / 8), b1 = q0 + (int)((int64_t)(q1 - q0) * (warp + 1) / 8);
    double gp = 0.0;
    // 32 partials at a time: one coalesced load of their flags, a ballot, then the valid ones in
    // ascending b, 8 independent loads per round trip (adding +0.0 for the unused slots)
    for (int c0 = b0; c0 < b1; c0 += 32) {
      const int cn = min(32, b1 - c0);
      unsigned mask;
      if (part_valid) mask = __ballot_sync(0xffffffffu, lane < cn && part_valid[c0 + lane] != 0);
      else mask = cn == 32 ? 0xffffffffu : ((1u << cn) - 1u);
      while (mask) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int bit = mask ? __ffs(mask) - 1 : -1;
          mask &= mask - 1u;
          v[u] = (bit >= 0 && k < m) ? part_vec[(size_t)(c0 + bit) * m + k] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) gp += v[u];
      }
    }
    red[warp][lane] = gp;
    __syncthreads();
    if (warp == 0) {
      double t = red[0][lane];
      for (int wi = 1; wi < 8; ++wi) t += red[wi][lane];
      gsum[lane] = t;
    }
    cg::cluster_group cluster = cg::this_cluster();
    cluster.sync();
    if (cs == 0 && warp == 0) {
      double t = gsum[lane];
      for (int q = 1; q < kEvalCS; ++q) t += cluster.map_shared_rank(gsum, q)[lane];
      red[0][lane] = t;
    }
    cluster.sync();  // rank 0 has read every CTA's sums
  }
  if (cs == 1 && rb == 0) {  // the scalar partials of K1/K1e, while the row blocks finish
    if (warp != 0) return false;
    double s[4] = {0, 0, 0, 0};
    for (int q0 = lane; q0 < nscal; q0 += 32 * 8) {  // lane sums q ≡ lane (mod 32) ascending; 8 in flight
      double v[8][4];
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int j = 0; j < 4; ++j) v[u][j] = q0 + 32 * u < nscal ? __ldcg(part_scal + (q0 + 32 * u) * 4 + j) : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int j = 0; j < 4; ++j) s[j] += v[u][j];
    }
    for (int j = 0; j < 4; ++j) s[j] = warp_allsum(s[j]);
    if (lane == 0) {
      for (int j = 0; j < 4; ++j) blk[nrb * 3 + j] = s[j];
      __threadfence();
      const unsigned t = atomicAdd(ticket, 1u);
      last = (t == (unsigned)nrb);
    }
    __syncwarp();
    if (!last) return false;
  }
  if (cs > 1 || (cs == 1 && rb != 0)) return false;
  if (cs == 0) {
  __syncthreads();
  if (warp == 0) {
    double yy = 0.0, by = 0.0, gg = 0.0;
    if (k < m) {
      yy = yk * yk;
      by = bk * yk;
      if (with_grad) {
        const double gp = red[0][lane];
        const double g = __dsub_rn(__dadd_rn(yk, bk), gp);
        g_out[k] = g;
        gg = g * g;
      }
    }
    yy = warp_allsum(yy);
    by = warp_allsum(by);
    gg = warp_allsum(gg);
    if (lane == 0) {
      blk[rb * 3 + 0] = yy;
      blk[rb * 3 + 1] = by;
      blk[rb * 3 + 2] = gg;
      __threadfence();
      const unsigned t = atomicAdd(ticket, 1u);
      last = (t == (unsigned)nrb);  // nrb row blocks + the scalar CTA
    }
  }
  __syncthreads();
  if (!last || warp != 0) return false;
  }
  __threadfence();
  // warp 0 of the last CTA: lane ℓ sums entries q ≡ ℓ (mod 32) in order, then a fixed butterfly
  double a = 0, bb = 0, c = 0;
  for (int q = lane; q < nrb; q += 32) {
    a += __ldcg(blk + q * 3 + 0);
    bb += __ldcg(blk + q * 3 + 1);
    c += __ldcg(blk + q * 3 + 2);
  }
  double s[4];
  for (int j = 0; j < 4; ++j) s[j] = __ldcg(blk + nrb * 3 + j);  // summed by CTA (0, 1)
  a = warp_allsum(a);
  bb = warp_allsum(bb);
  c = warp_allsum(c);
  if (lane != 0) return false;
  EvalOut o;
  o.yy = a;
  o.by = bb;
  o.gg = c;
  for (int j = 0; j < 4; ++j) o.s[j] = s[j];
  const double tprox = __dmul_rn(sc.cpsi, s[0]);
  o.psi = __dadd_rn(__dadd_rn(__dmul_rn(0.5, a), bb), tprox);
  o.psimag = fabs(0.5 * a) + fabs(bb) + fabs(tprox);
  o.res1 = with_grad ? sqrt(c) / (1.0 + nb) : -1.0;
  o.gd = gd_src ? *gd_src : 0.0;
  o.r = r_in ? (long long)*r_in : -1;
  o.info = info_src ? (long long)*info_src : 0;
  o.seq = seq;
  o.pad = 0;
  *out = o;
  if (host_out) {  // zero-copy to mapped pinned memory; seq last, after a system-scope fence
    volatile EvalOut* h = host_out;
    h->psi = o.psi; h->psimag = o.psimag; h->res1 = o.res1; h->yy = o.yy; h->by = o.by; h->gg = o.gg;
    for (int j = 0; j < 4; ++j) h->s[j] = o.s[j];
    h->gd = o.gd; h->r = o.r; h->info = o.info;
    __threadfence_system();
    h->seq = seq;
  }
  *ticket = 0u;  // ready for the next launch (stream-ordered)
  return true;  // the finishing thread (EvalOut written)
}

// m ≤ 512: ONE 16-CTA cluster, CTA q = row block q.  Its 8 warps split the partial rows (contiguous
// eighths, ascending b, the same ballot / 8-in-flight loads), the warp sums are added in warp order,
// the block's (yyᵀ, bᵀy, gᵀg) pieces go to rank 0's shared memory through DSMEM while rank 1 sums
// the K1 scalar partials; after one cluster barrier rank 0 adds the blocks in order and writes
// EvalOut.  No global ticket, no second reduction level.  True on rank 0, thread 0.
constexpr int kEval16 = 16;
SSN_DEV bool eval_body16(int64_t m, const double* __restrict__ y, const double* __restrict__ bvec,
                         const double* __restrict__ part_vec, const int* __restrict__ part_valid, int nparts,
                         const double* __restrict__ part_scal, int nscal, Scal sc, double nb, int with_grad,
                         double* __restrict__ g_out, const int64_t* r_in, EvalOut* out, const double* gd_src,
                         const int* info_src, EvalOut* host_out, unsigned long long seq, const Scal* scp,
                         const int* pred, const double* nbp) {
  __shared__ double red[8][33];
  __shared__ double bsum[kEval16 * 3 + 4];  // rank 0: per-block (yy, by, gg), then the 4 scalar sums
  if (pred && *pred == 0) return false;  // graph mode: predicated off (uniform over the cluster)
  if (scp) sc = *scp;
  if (nbp) nb = *nbp;
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = (int)cluster.block_rank();
  const int64_t k = (int64_t)q * 32 + lane;
  double yk = 0.0, bk = 0.0;
  if (warp == 0 && k < m) {
    yk = y[k];
    bk = bvec[k];
  }
  double gp = 0.0;
  if (with_grad) {
    const int b0 = (int)((int64_t)nparts * warp / 8), b1 = (int)((int64_t)nparts * (warp + 1) / 8);
    for (int c0 = b0; c0 < b1; c0 += 32) {
      const int cn = min(32, b1 - c0);
      unsigned mask;
      if (part_valid) mask = __ballot_sync(0xffffffffu, lane < cn && part_valid[c0 + lane] != 0);
      else mask = cn == 32 ? 0xffffffffu : ((1u << cn) - 1u);
      while (mask) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int bit = mask ? __ffs(mask) - 1 : -1;
          mask &= mask - 1u;
          v[u] = (bit >= 0 && k < m) ? part_vec[(size_t)(c0 + bit) * m + k] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) gp += v[u];
      }
    }
    red[warp][lane] = gp;
  }
  __syncthreads();
  if (warp == 0) {
    double yy = 0.0, by = 0.0, gg = 0.0;
    if (k < m) {
      yy = yk * yk;
      by = bk * yk;
      if (with_grad) {
        double t = red[0][lane];
        for (int wi = 1; wi < 8; ++wi) t += red[wi][lane];
        const double g = __dsub_rn(__dadd_rn(yk, bk), t);
        g_out[k] = g;
        gg = g * g;
      }
    }
    yy = warp_allsum(yy);
    by = warp_allsum(by);
    gg = warp_allsum(gg);
    if (lane == 0) {
      double* dst = cluster.map_shared_rank(bsum, 0);
      dst[q * 3 + 0] = yy;
      dst[q * 3 + 1] = by;
      dst[q * 3 + 2] = gg;
    }
  } else if (q == 1 && warp == 1) {  // the scalar partials of K1/K1e (lane sums q' ≡ lane mod 32, 8 in flight)
    double s[4] = {0, 0, 0, 0};
    for (int q0 = lane; q0 < nscal; q0 += 32 * 8) {
      double v[8][4];
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int j = 0; j < 4; ++j) v[u][j] = q0 + 32 * u < nscal ? __ldcg(part_scal + (q0 + 32 * u) * 4 + j) : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int j = 0; j < 4; ++j) s[j] += v[u][j];
    }
    for (int j = 0; j < 4; ++j) s[j] = warp_allsum(s[j]);
    if (lane == 0) {
      double* dst = cluster.map_shared_rank(bsum, 0);
      for (int j = 0; j < 4; ++j) dst[kEval16 * 3 + j] = s[j];
    }
  }
  cluster.sync();  // every block's pieces are in rank 0's shared memory
  if (q != 0 || tid != 0) return false;
  const int nrb = (int)((m + 31) / 32);
  double a = 0, bb = 0, c = 0;
  for (int qq = 0; qq < nrb; ++qq) {
    a += bsum[qq * 3 + 0];
    bb += bsum[qq * 3 + 1];
    c += bsum[qq * 3 + 2];
  }
  double s4[4];
  for (int j = 0; j < 4; ++j) s4[j] = bsum[kEval16 * 3 + j];
  EvalOut o;
  o.yy = a;
  o.by = bb;
  o.gg = c;
  for (int j = 0; j < 4; ++j) o.s[j] = s4[j];
  const double tprox = __dmul_rn(sc.cpsi, s4[0]);
  o.psi = __dadd_rn(__dadd_rn(__dmul_rn(0.5, a), bb), tprox);
  o.psimag = fabs(0.5 * a) + fabs(bb) + fabs(tprox);
  o.res1 = with_grad ? sqrt(c) / (1.0 + nb) : -1.0;
  o.gd = gd_src ? *gd_src : 0.0;
  o.r = r_in ? (long long)*r_in : -1;
  o.info = info_src ? (long long)*info_src : 0;
  o.seq = seq;
  o.pad = 0;
  *out = o;
  if (host_out) {  // zero-copy to mapped pinned memory; seq last, after a system-scope fence
    volatile EvalOut* h = host_out;
    h->psi = o.psi; h->psimag = o.psimag; h->res1 = o.res1; h->yy = o.yy; h->by = o.by; h->gg = o.gg;
    for (int j = 0; j < 4; ++j) h->s[j] = o.s[j];
    h->gd = o.gd; h->r = o.r; h->info = o.info;
    __threadfence_system();
    h->seq = seq;
  }
  return true;
}

__global__ void __cluster_dims__(kEval16, 1, 1) __launch_bounds__(K5_THREADS)
    k_eval_reduce16(int64_t m, const double* __restrict__ y, const double* __restrict__ bvec,
                    const double* __restrict__ part_vec, const int* __restrict__ part_valid, int nparts,
                    const double* __restrict__ part_scal, int nscal, Scal sc, double nb, int with_grad,
                    double* __restrict__ g_out, const int64_t* r_in, EvalOut* out, double* blk, unsigned* ticket,
                    const double* gd_src, const int* info_src, EvalOut* host_out, unsigned long long seq,
                    const Scal* scp, const int* pred, const double* nbp) {
  eval_body16(m, y, bvec, part_vec, part_valid, nparts, part_scal, nscal, sc, nb, with_grad, g_out, r_in, out, gd_src,
              info_src, host_out, seq, scp, pred, nbp);
}

__global__ void __cluster_dims__(kEvalCS, 1, 1) __launch_bounds__(K5_THREADS) k_eval_reduce(int64_t m, const double* __restrict__ y,
                                                            const double* __restrict__ bvec,
                                                            const double* __restrict__ part_vec,
                                                            const int* __restrict__ part_valid, int nparts,
                                                            const double* __restrict__ part_scal, int nscal,
                                                            Scal sc, double nb, int with_grad,
                                                            double* __restrict__ g_out, const int64_t* r_in,
                                                            EvalOut* out, double* blk, unsigned* ticket,
                                                            const double* gd_src, const int* info_src,
                                                            EvalOut* host_out, unsigned long long seq,
                                                            const Scal* scp, const int* pred, const double* nbp) {
  eval_body(m, y, bvec, part_vec, part_valid, nparts, part_scal, nscal, sc, nb, with_grad, g_out, r_in, out, blk,
            ticket, gd_src, info_src, host_out, seq, scp, pred, nbp);
}

// max over G plain-mode partials (λmax = ‖Aᵀb‖∞)
// R40 gate: the reused-Aᵀb launch of K1 reads the active columns of A from global memory for the ∇ψ
// partial rows, so it only pays while the first trial's active set {i : |Aᵀb|_i > λ1} (x = 0) is small.
// Counts it and sets *flag = (count ≤ limit).  A heuristic only: both K1 modes write the same bits.
// cnt[0] = count, cnt[1] = ticket; both zero on entry and on exit.
__global__ void __launch_bounds__(256) k_atb_gate(const double* __restrict__ atb, int64_t n, double l1, int64_t limit,
                                                  unsigned long long* cnt, int* flag, int* flag2) {
  unsigned long long c = 0;
  for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256)
    c += fabs(atb[i]) > l1;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  __shared__ unsigned long long sw[8];
  if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < 8; ++w) t += sw[w];
    atomicAdd(cnt, t);
    __threadfence();
    if (atomicAdd(cnt + 1, 1ull) == gridDim.x - 1) {
      const unsigned long long tot = atomicAdd(cnt, 0ull);
      const int f = tot <= (unsigned long long)limit;
      *flag = f;
      if (flag2) *flag2 = f;
      cnt[0] = 0ull;
      cnt[1] = 0ull;
    }
  }
}

__global__ void k_max_partials(const double* part_scal, int G, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double v = 0.0;
    for (int q = 0; q < G; ++q) v = fmax(v, part_scal[q * 4]);
    *out = v;
  }
}

}  // namespace ssn
