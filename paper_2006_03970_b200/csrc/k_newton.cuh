// k_newton.cuh — the generalized-Hessian system V d = −∇ψ, V = I_m + κ A_J A_Jᵀ
// (Eq. (16)-(18)), with the Sherman–Morrison–Woodbury form Eq. (19)
// when r < m.  All products read the active columns A[:, J[a]] in place
// (each column is m contiguous doubles); nothing is gathered into a copy.
//
// K2  k_gather_axpy    : per-CTA partials of Σ_a coef_a A[:, J_a]          (A_J v, A_J P_J)
//     k_gather_rows    : row-block clusters: A_J coef (∇ψ) or d = −g + A_J v, gᵀd, y + d (SMW)
//     k_combine        : out = bs·base + Σ parts (fixed order), optional dot
// K3  k_gram<true>     : split-K partials of A_JᵀA_J (lower, r × r) and u = A_Jᵀg Eq. (19)
//     k_gram<false>    : split-K partials of A_J A_Jᵀ (lower, m × m)            Eq. (18)
//     k_gram_reduce    : κ⁻¹ I_r + Σ  /  I_m + κ Σ
// K4  k_chol_cluster   : Cholesky by one thread-block cluster with the forward solve carried
//                        as an extra matrix row and a block backward solve (one launch)
#pragma once
#include <cooperative_groups.h>
#include <type_traits>
#include "common.cuh"

namespace ssn {

// ---------------------------------------------------------------------------
// Geometry of the Newton direction for an active set of size r (Eq. (18) / (19)).  Computed by
// the same function on the host (host-driven mode) and on the device (graph mode), so both
// modes launch identical work decompositions and produce bitwise-identical results.
// ---------------------------------------------------------------------------
struct DirGeo {
  int branch;          // 0: r = 0 (d = −g), 1: 0 < r < m (SMW, Eq. (19)), 2: r ≥ m (Eq. (18)), 3: CG (R32)
  int N, NR, ld;       // factor order, rows incl. the rhs row, leading dimension of Mmat
  int tiles, ns;       // Gram lower 32 × 32 tiles and split-K slices
  int pad0;
  int pad;
  long long r, nout, nmat;
  double diag, mult;   // reduce: M = diag·I + mult·Σ_s W[s]; CG: mult = κ
  double jit;          // factor retry (R36): M_ii ← M_ii (1 + jit); 0 on a first attempt
};

// Strategy (R12, R32): CG iff r > cg_ratio·m (cg_ratio > 0) or min(m, r) > cg_threshold.
SSN_HD bool use_cg(long long r, long long m, double cg_ratio, double cg_threshold) {
  const long long mn = r < m ? r : m;
  return r > 0 && ((cg_ratio > 0.0 && (double)r > cg_ratio * (double)m) || (double)mn > cg_threshold);
}

// K3 Gram: lower 64 × 64 output tiles of an nout × nout matrix
constexpr int GT = 64;  // Gram output tile edge
SSN_HD int gram_tiles(long long nout) {
  const int nt = (int)((nout + GT - 1) / GT);
  return nt * (nt + 1) / 2;
}

// split-K slices: enough (tile, slice) items to cover 2 CTAs per SM, ≤ one slice per 32-chunk
SSN_HD int gram_splits(int nsm, int tiles, long long K, int wsplits) {
  int ns = (2 * nsm + tiles - 1) / tiles;
  const long long nch = (K + 31) / 32;
  if (ns > nch) ns = (int)nch;
  if (ns > wsplits) ns = wsplits;
  return ns < 1 ? 1 : ns;
}

SSN_HD DirGeo make_geo(long long r, long long m, int nsm, int wsplits, double kappa, double kinv, double cg_ratio,
                       double cg_threshold) {
  DirGeo g;
  g.r = r;
  g.pad0 = g.pad = 0;
  g.jit = 0.0;
  if (use_cg(r, m, cg_ratio, cg_threshold)) {
    g.branch = 3;
    g.N = g.NR = g.ld = g.tiles = g.ns = 0;
    g.nout = g.nmat = 0;
    g.diag = 0.0;
    g.mult = kappa;
  } else if (r == 0) {
    g.branch = 0;
    g.N = g.NR = g.ld = g.tiles = g.ns = 0;
    g.nout = g.nmat = 0;
    g.diag = g.mult = 0.0;
  } else if (r < m) {
    g.branch = 1;
    g.N = (int)r;
    g.NR = g.N + 1;
    g.ld = g.N + 1;
    g.nout = r + 1;  // index r carries g: row r = u = A_Jᵀg (the rhs row)
    g.nmat = r;
    g.tiles = gram_tiles(g.nout);
    g.ns = gram_splits(nsm, g.tiles, m, wsplits);
    g.diag = kinv;  // κ⁻¹ I_r + A_JᵀA_J (R13)
    g.mult = 1.0;
  } else {
    g.branch = 2;
    g.N = (int)m;
    g.NR = g.N + 1;
    g.ld = g.N + 1;
    g.nout = g.nmat = m;
    g.tiles = gram_tiles(m);
    g.ns = gram_splits(nsm, g.tiles, r, wsplits);
    g.diag = 1.0;  // I_m + κ A_J A_Jᵀ
    g.mult = kappa;
  }
  return g;
}

// ---------------------------------------------------------------------------
// K2: part_vec[b][k] = Σ_{a ∈ chunk b} coef[a] * A[k, J[a]]
// ---------------------------------------------------------------------------
// r is read from r_dev when r < 0 (device-resident count, fixed grid); valid[b] (nullable)
// records whether CTA b had any column, so empty CTAs skip writing their partial row.
template <class Acc, int MR>
__global__ void __launch_bounds__(256) k_gather_axpy(const Acc A, int64_t m,
                                                     const int32_t* __restrict__ J, const double* __restrict__ coef,
                                                     int64_t r, const int64_t* __restrict__ r_dev,
                                                     double* __restrict__ part_vec, int* __restrict__ valid,
                                                     const int* __restrict__ pred) {
  extern __shared__ double red[];  // 8 x m
  if (pred && *pred == 0) return;  // graph mode: predicated off (the consumer is predicated too)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool devr = r < 0;
  if (devr) r = *r_dev;
  // host r: contiguous share; device r: chunks of 16 columns b, b + grid, ... (few CTAs for small r)
  const int64_t a_lo = devr ? (int64_t)blockIdx.x * 16 : (int64_t)blockIdx.x * r / gridDim.x;
  const int64_t a_hi = devr ? r : (int64_t)(blockIdx.x + 1) * r / gridDim.x;
  if (valid && threadIdx.x == 0) valid[blockIdx.x] = a_hi > a_lo;
  if (valid && a_hi <= a_lo) return;
  double acc[MR];
#pragma unroll
  for (int t = 0; t < MR; ++t) acc[t] = 0.0;
  const int64_t stride = devr ? (int64_t)gridDim.x * 16 : 0;
  for (int64_t base = a_lo; base < a_hi; base += stride) {
    const int64_t e_hi = devr ? min(base + 16, a_hi) : a_hi;
    for (int64_t a = base + warp; a < e_hi; a += 8) {
      const auto col = A.col(J[a]);
      const double c = coef[a];
#pragma unroll
      for (int t = 0; t < MR; ++t) {
        const int64_t row = lane + 32 * t;
        if (row < m) acc[t] = fma(c, col.ld(row), acc[t]);
      }
    }
    if (!devr) break;
  }
#pragma unroll
  for (int t = 0; t < MR; ++t) {
    const int64_t row = lane + 32 * t;
    if (row < m) red[(size_t)warp * m + row] = acc[t];
  }
  __syncthreads();
  for (int64_t k = threadIdx.x; k < m; k += blockDim.x) {
    double v = red[k];
    for (int wi = 1; wi < 8; ++wi) v += red[(size_t)wi * m + k];
    part_vec[(size_t)blockIdx.x * m + k] = v;
  }
}

// K2 by row blocks (the hot gathers): lane ℓ of every warp owns row k = 32·rb + ℓ of the row block
// rb = cluster index; the 8 CTAs of a cluster split the r columns in 8 contiguous ranges, each
// CTA stages its J / coef in smem and its warps issue 8 independent column loads per round trip.
// The cluster's rank-0 CTA sums the 8 per-CTA partials through DSMEM in rank order, so one
// launch yields the finished m-vector (no partial vectors in HBM, no second kernel):
//   kGatherVec: out = Σ_a coef_a A[:, J_a]                      (∇ψ's A_J P_J, Eq. (15))
//   kGatherSmw: out = d = −g + Σ_a v_a A[:, J_a], yt = y + d, *gd_out = gᵀd   (Eq. (19))
// r: host value (≥ 0), else *r_dev; graph mode: pred (nullable) / geo (SMW branch) predicate.
constexpr int kGatherCS = 8;  // cluster size = column splits per row block
enum { kGatherVec = 0, kGatherSmw = 1 };
template <class Acc>
__global__ void __cluster_dims__(kGatherCS, 1, 1) __launch_bounds__(256)
    k_gather_rows(const Acc A, int64_t m, const int32_t* __restrict__ J, const double* __restrict__ coef, int64_t r,
                  const int64_t* __restrict__ r_dev, const int* __restrict__ pred, const DirGeo* geo, int mode,
                  double* __restrict__ out, const double* __restrict__ g, const double* __restrict__ y,
                  double* __restrict__ yt, double* gd_out, double* gdpart, unsigned* ticket) {
  __shared__ int32_t sJ[256];
  __shared__ double sC[256];
  __shared__ double red[8][32];
  __shared__ double part[32];
  __shared__ bool last;
  if (pred && *pred == 0) return;  // uniform over the grid
  if (geo) {  // SMW back-substitution (branch 1), or d = −g for r = 0 (branch 0: no columns)
    if (geo->branch != 1 && geo->branch != 0) return;
    r = geo->branch == 1 ? geo->r : 0;
  } else if (r < 0) {
    r = *r_dev;
  }
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cs = (int)cluster.block_rank();
  const int rb = (int)(blockIdx.x / kGatherCS);
  const int64_t row = (int64_t)rb * 32 + lane;
  const int64_t lo = r * cs / kGatherCS, hi = r * (cs + 1) / kGatherCS;
  double acc = 0.0;
  for (int64_t c0 = lo; c0 < hi; c0 += 256) {
    const int cn = (int)min((int64_t)256, hi - c0);
    if (tid < cn) {
      sJ[tid] = J[c0 + tid];
      sC[tid] = coef[c0 + tid];
    }
    __syncthreads();
    for (int e0 = warp; e0 < cn; e0 += 64) {  // this warp: columns e0, e0 + 8, …, e0 + 56
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + 8 * u;
        v[u] = (e < cn && row < m) ? A.col(sJ[e]).ld(row) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + 8 * u;
        if (e < cn) acc = fma(sC[e], v[u], acc);
      }
    }
    __syncthreads();
  }
  red[warp][lane] = acc;
  __syncthreads();
  if (warp == 0) {
    double t = red[0][lane];
    for (int wi = 1; wi < 8; ++wi) t += red[wi][lane];
    part[lane] = t;
  }
  cluster.sync();
  if (cs == 0 && warp == 0) {
    double tot = part[lane];
    for (int q = 1; q < kGatherCS; ++q) tot += cluster.map_shared_rank(part, q)[lane];
    if (mode == kGatherVec) {
      if (row < m) out[row] = tot;
    } else {
      double dot = 0.0;
      if (row < m) {
        const double dk = -g[row] + tot;
        out[row] = dk;
        yt[row] = __dadd_rn(y[row], dk);
        dot = g[row] * dk;
      }
      dot = warp_allsum(dot);
      if (lane == 0) {
        gdpart[rb] = dot;
        __threadfence();
        last = atomicAdd(ticket, 1u) == (unsigned)(gridDim.x / kGatherCS) - 1;
      }
      __syncwarp();
      if (last && lane == 0) {  // gᵀd = Σ_rb partials in row-block order
        __threadfence();
        double sdot = 0.0;
        for (unsigned q = 0; q < gridDim.x / kGatherCS; ++q) sdot += __ldcg(gdpart + q);
        *gd_out = sdot;
        *ticket = 0u;
      }
    }
  }
  cluster.sync();  // the partials stay resident until rank 0 has read them
}

// out[k] = bs*base[k] + Σ_{b<nparts} parts[b][k] (b ascending); if dotv: *dot_out = Σ dotv·out
__global__ void __launch_bounds__(1024) k_combine(int64_t m, const double* __restrict__ base, double bs,
                                                  const double* __restrict__ parts, int nparts,
                                                  double* __restrict__ out, const double* __restrict__ dotv,
                                                  double* dot_out, const int* __restrict__ valid) {
  __shared__ double red[32];
  const int tid = threadIdx.x;
  double dot = 0.0;
  for (int64_t k = tid; k < m; k += blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nparts; ++b)
      if (!valid || valid[b]) s += parts[(size_t)b * m + k];
    const double v = (base ? bs * base[k] : 0.0) + s;
    out[k] = v;
    if (dotv) dot += dotv[k] * v;
  }
  if (dotv) {
    dot = warp_allsum(dot);
    if ((tid & 31) == 0) red[tid >> 5] = dot;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int wi = 0; wi < (int)(blockDim.x >> 5); ++wi) s += red[wi];
      *dot_out = s;
    }
  }
}

// ---------------------------------------------------------------------------
// K3: Gram builds, 32x32 output tile per CTA, 256 threads (4 outputs each)
// ---------------------------------------------------------------------------
SSN_DEV void tri_tile(int q, int* ti, int* tj) {  // q → (ti ≥ tj), row-major over lower tiles
  int i = (int)((sqrt(8.0 * q + 1.0) - 1.0) * 0.5);
  while ((i + 1) * (i + 2) / 2 <= q) ++i;
  while (i * (i + 1) / 2 > q) --i;
  *ti = i;
  *tj = q - i * (i + 1) / 2;
}

// M[i + j*ld] = diag·[i == j] + mult · Σ_s W[s][i + j*nout]   (i ≥ j, j < nmat)
//   retry after a failed factor (R36): M_ii ← M_ii + jit·M_ii
//   SMW:   diag = κ⁻¹, mult = 1; nout = nmat + 1: row nmat is the rhs u = A_Jᵀg (unscaled)
//   m × m: diag = 1, mult = κ (oracle: κ s + δ); nout = nmat; rhs row ← g (if g)
// Grid-stride; graph mode reads the sizes from the device geometry (predicated on the branch).
__global__ void k_gram_reduce(const double* __restrict__ W, int ns, int64_t nout, int64_t nmat, double diag,
                              double mult, double* __restrict__ M, int64_t ld, const double* __restrict__ g,
                              const DirGeo* geo, int want, double jit) {
  if (geo) {  // want < 0: either exact branch (the rhs row g only for r ≥ m)
    if (want >= 0 ? geo->branch != want : (geo->branch != 1 && geo->branch != 2)) return;
    if (want < 0 && geo->branch != 2) g = nullptr;
    ns = geo->ns;
    nout = geo->nout;
    nmat = geo->nmat;
    diag = geo->diag;
    mult = geo->mult;
    ld = geo->ld;
    jit = geo->jit;
  }
  const int64_t tot = nout * nout > nmat ? nout * nout : nmat;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    if (g && e < nmat) M[nmat + e * ld] = g[e];
    if (e >= nout * nout) continue;
    const int64_t i = e % nout, j = e / nout;
    if (i < j || j >= nmat) continue;
    double s = 0.0;
    for (int q = 0; q < ns; ++q) s += W[(size_t)q * nout * nout + e];
    if (i < nmat) {
      double v = (mult == 1.0 ? s : mult * s) + (i == j ? diag : 0.0);
      if (i == j && jit != 0.0) v = __fma_rn(v, jit, v);
      M[i + j * ld] = v;
    } else {
      M[i + j * ld] = s;  // rhs row
    }
  }
}

// ---------------------------------------------------------------------------
// K4: SPD solve by one thread-block cluster (Cholesky, right-looking, 32 × 32 tiles in L2).
//
// M is NR × N column-major with ld ≥ NR: rows 0..N-1 hold the SPD matrix (lower triangle used
// and overwritten by L), rows N..NR-1 are appended rows C that leave the factorisation as
// C L⁻ᵀ; with `out` row N is the right-hand side, so the factorisation performs the forward
// substitution z = L⁻¹ rhs for free.  Per panel k (W_k = L_kk⁻¹ already in Winv):
//   B: L_ik = A_ik W_kᵀ for row tiles i > k (appended rows included) — DMMA tile GEMM, warp/tile
//      | cluster barrier
//   C: A_ij −= L_ik L_jkᵀ for k < j ≤ i                                — DMMA tile GEMM, warp/tile
//      look-ahead: CTA 0 warps 0-3 update tile (k+1,k+1) into smem, then warp 0 factors it and
//      inverts it in one register-resident sweep (W_{k+1}); the other warps take the rest
//      | cluster barrier
// Then CTA 0 runs the backward substitution v = L⁻ᵀ z right-looking over the blocks.
// FP64 tensor cores: mma.sync.m8n8k4.f64 (SASS DMMA) — the tile updates are dense contractions.
// out = scale · v; if dotv: *dot_out = Σ dotv · out; if yt: yt = ybase + out.
// ---------------------------------------------------------------------------
// Per-branch outputs of a K4 launch that serves both exact branches (graph mode, want < 0):
// [0] SMW (v → u), [1] m × m (d = −M⁻¹g, gᵀd, y + d)
struct CholArgs {
  double* out;
  double scale;
  const double* dotv;
  double* dot_out;
  const double* ybase;
  double* yt;
};

constexpr int CHT = 32;  // tile edge
constexpr int TLD = 33;  // smem tile leading dimension
constexpr int kColSlots = 3;  // column tiles a worker quad holds for the TRSM (≤ 3 × 30 quads ≥ 64 row tiles)

SSN_DEV void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// One warp's 8 × 32 strip of a 32 × 32 × 32 product: acc[cb] += sgn · Σ_p SA[8w + g][p] SB[8cb + ·][p].
// DMMA latency is ~270 cycles (tools/probes/mma_probe), so the K loop is split over 4 accumulator
// groups (16 independent chains instead of 4), summed at the end.
SSN_DEV void strip_mma(const double* SA, const double* SB, double (&acc)[4][2], double sgn, int w, int lane) {
  const int g = lane >> 2, t = lane & 3;
  double part[4][4][2];
#pragma unroll
  for (int h = 0; h < 4; ++h)
#pragma unroll
    for (int cb = 0; cb < 4; ++cb) part[h][cb][0] = part[h][cb][1] = 0.0;
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    const int h = kk & 3;
    const double af = sgn * SA[(8 * w + g) * TLD + 4 * kk + t];
#pragma unroll
    for (int cb = 0; cb < 4; ++cb) dmma(part[h][cb], af, SB[(8 * cb + g) * TLD + 4 * kk + t]);
  }
#pragma unroll
  for (int cb = 0; cb < 4; ++cb)
#pragma unroll
    for (int e = 0; e < 2; ++e) acc[cb][e] += (part[0][cb][e] + part[1][cb][e]) + (part[2][cb][e] + part[3][cb][e]);
}

// acc[rb][cb] += sgn · Σ_p SA[r][p] · SB[c][p] over a 32 × 32 × 32 tile (rows r = 8rb + lane/4,
// cols c = 8cb + 2(lane%4) + e in the C fragment layout of m8n8k4).
SSN_DEV void tile_mma(const double* SA, const double* SB, double (&acc)[4][4][2], double sgn, int lane) {
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    double af[4], bf[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      af[b] = sgn * SA[(8 * b + g) * TLD + 4 * kk + t];
      bf[b] = SB[(8 * b + g) * TLD + 4 * kk + t];
    }
#pragma unroll
    for (int rb = 0; rb < 4; ++rb)
#pragma unroll
      for (int cb = 0; cb < 4; ++cb) dmma(acc[rb][cb], af[rb], bf[cb]);
  }
}

// K3: split-K Gram tiles on the FP64 tensor cores.  64 × 64 output tiles; the reduction runs in
// 32-chunks staged through shared memory (register double buffer), 8 warps × (16 × 32) blocks of
// m8n8k4 DMMAs (8 independent accumulator chains per warp).  Operand element (output idx ω, κ):
//   SMW   (Eq. (19)): out(a, b) = Σ_k A[k,J_a] A[k,J_b];  ω = a, κ = k − 32·chunk; index r = g
//   m × m (Eq. (18)): out(k, l) = Σ_a A[k,J_a] A[l,J_a];  ω = k, κ = a − 32·chunk
// Shared layouts are chosen for conflict-free fragment reads and coalesced global loads: SMW
// [ω][κ] (ld 36: a warp loads one column's 32 consecutive rows), m × m [κ][ω] (ld 68: a warp
// loads 64 consecutive rows of one column).  Work items (lower tile q, slice s), item = q + tiles·s,
// are taken by persistent CTAs in a grid-stride loop (results do not depend on the grid); each
// writes its partial tile (lower part) to W[s] and k_gram_reduce sums the slices in order.
// Graph mode: r, tiles, ns from the device geometry (predicated on the branch).
constexpr int kGramSmem = GT * 36;  // doubles per operand buffer (≥ 32 · 68 of the m × m layout)
// One (tile, K-slice) item: the 64 × 64 output tile (ti, tj) summed over reduction chunks
// [c_lo, c_hi) into this thread's fragment acc (rows 16wr + 8i + g, cols 32wc + 8j + 2t + e).
template <bool SMW, class Acc>
SSN_DEV void gram_item(const Acc& A, int64_t m, const int32_t* __restrict__ J, int64_t r,
                       const double* __restrict__ gext, int ti, int tj, int64_t c_lo, int64_t c_hi, double* sA,
                       double* sB, double (&acc)[2][4][2]) {
  constexpr int LD = SMW ? 36 : 68;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wr = warp >> 1, wc = warp & 1;  // this warp's block: rows 16 wr …, cols 32 wc …
  auto at = [&](int w, int k) { return SMW ? w * LD + k : k * LD + w; };
  const bool dg = ti == tj;
  const int64_t o0 = (int64_t)ti * GT, o1 = (int64_t)tj * GT;
  double va[8], vb[8];
  // SMW: value q is (ω = warp + 8q, κ = lane); m × m: (ω = lane + 32(q & 1), κ = warp + 8(q >> 1))
  auto load = [&](int64_t ch) {
    if (SMW) {
      const int64_t k = ch * 32 + lane;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int64_t a = o0 + warp + 8 * q, b = o1 + warp + 8 * q;
        va[q] = k >= m ? 0.0 : (a < r ? A.col(J[a]).ld(k) : ((a == r && gext) ? __ldg(gext + k) : 0.0));
        vb[q] = (dg || k >= m) ? 0.0 : (b < r ? A.col(J[b]).ld(k) : ((b == r && gext) ? __ldg(gext + k) : 0.0));
      }
    } else {
#pragma unroll
      for (int q2 = 0; q2 < 4; ++q2) {
        const int64_t a = ch * 32 + warp + 8 * q2;
        const bool ok = a < r;
        const auto col = A.col(ok ? (int64_t)J[a] : 0);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t ra = o0 + lane + 32 * h, rb = o1 + lane + 32 * h;
          va[2 * q2 + h] = (ok && ra < m) ? col.ld(ra) : 0.0;
          vb[2 * q2 + h] = (ok && !dg && rb < m) ? col.ld(rb) : 0.0;
        }
      }
    }
  };
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  if (c_lo < c_hi) load(c_lo);
  for (int64_t ch = c_lo; ch < c_hi; ++ch) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int w = SMW ? warp + 8 * q : lane + 32 * (q & 1);
      const int k = SMW ? lane : warp + 8 * (q >> 1);
      sA[at(w, k)] = va[q];
      if (!dg) sB[at(w, k)] = vb[q];
    }
    __syncthreads();
    if (ch + 1 < c_hi) load(ch + 1);
    const double* SB = dg ? sA : sB;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      double af[2], bf[4];
#pragma unroll
      for (int i = 0; i < 2; ++i) af[i] = sA[at(16 * wr + 8 * i + g, 4 * kk + t)];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = SB[at(32 * wc + 8 * j + g, 4 * kk + t)];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], af[i], bf[j]);
    }
    __syncthreads();
  }
}

template <bool SMW, class Acc>
SSN_DEV void gram_body(const Acc& A, int64_t m, const int32_t* __restrict__ J, int64_t r, double* __restrict__ W,
                       const double* __restrict__ gext, int tiles, int ns, double* sA, double* sB) {
  const int64_t K = SMW ? m : r;  // reduction length
  const int64_t nch = (K + 31) / 32;
  const int64_t nout = SMW ? r + (gext ? 1 : 0) : m;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wr = warp >> 1, wc = warp & 1;
  for (int item = blockIdx.x; item < tiles * ns; item += gridDim.x) {
    int ti, tj;
    tri_tile(item % tiles, &ti, &tj);
    const int s = item / tiles;
    const int64_t o0 = (int64_t)ti * GT, o1 = (int64_t)tj * GT;
    double acc[2][4][2];
    gram_item<SMW>(A, m, J, r, gext, ti, tj, nch * s / ns, nch * (s + 1) / ns, sA, sB, acc);
    double* Ws = W + (size_t)s * nout * nout;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t oi = o0 + 16 * wr + 8 * i + g, oj = o1 + 32 * wc + 8 * j + 2 * t + e;
          if (oi < nout && oj < nout && oi >= oj) Ws[oi + oj * nout] = acc[i][j][e];
        }
  }
}

// K3 fused with its split-K reduction (the hot-path Newton systems, Eq. (18)/(19)): one 8-CTA
// cluster per 64 × 64 output tile, CTA rank s sums K-slice s; the 8 partial tiles meet in
// distributed shared memory and rank s reduces rows 8s … 8s + 7 in rank order (deterministic),
// applying the k_gram_reduce epilogue (× mult, + diag, jitter, right-hand-side row) straight into
// M.  No slice buffer in global memory and no second launch.  Clusters take tiles in a stride
// loop; graph mode reads the branch and sizes from the device geometry.
constexpr int kGramCS = 8;
struct GramFusedArgs {
  int branch;  // 1: SMW (Eq. (19), gext = g as the extra column r), 2: m × m (Eq. (18), g as rhs row)
  int64_t r, nout, nmat;
  int tiles, ld;
  double diag, mult, jit;
};
template <class Acc>
__global__ void __cluster_dims__(kGramCS, 1, 1) __launch_bounds__(256)
    k_gram_fused(const Acc A, int64_t m, const int32_t* __restrict__ J, double* __restrict__ M,
                 const double* __restrict__ g, GramFusedArgs ga, const DirGeo* geo, int only = 0) {
  __shared__ __align__(16) double sm[2 * kGramSmem];  // operand buffers, then the partial tile (64 × 65)
  if (geo) {  // only > 0: this branch alone (the sharded SMW form on the gathered columns)
    if ((geo->branch != 1 && geo->branch != 2) || (only && geo->branch != only)) return;
    ga.branch = geo->branch;
    ga.r = geo->r;
    ga.nout = geo->nout;
    ga.nmat = geo->nmat;
    ga.tiles = geo->tiles;
    ga.ld = geo->ld;
    ga.diag = geo->diag;
    ga.mult = geo->mult;
    ga.jit = geo->jit;
  }
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int s = (int)cluster.block_rank(), cl = (int)(blockIdx.x / kGramCS), ncl = (int)(gridDim.x / kGramCS);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, t = lane & 3, wr = warp >> 1, wc = warp & 1;
  const bool smw = ga.branch == 1;
  const int64_t K = smw ? m : ga.r;
  const int64_t nch = (K + 31) / 32;
  double* sA = sm;
  double* sB = sm + kGramSmem;
  double* Pt = sm;  // partial tile [64][65]
  if (!smw && g && cl == 0)  // the rhs row of Eq. (18): M[nmat + e·ld] = g[e]
    for (int64_t e = s * 256 + tid; e < ga.nmat; e += kGramCS * 256) M[ga.nmat + e * ga.ld] = g[e];
  for (int tq = cl; tq < ga.tiles; tq += ncl) {
    int ti, tj;
    tri_tile(tq, &ti, &tj);
    double acc[2][4][2];
    if (smw) gram_item<true>(A, m, J, ga.r, g, ti, tj, nch * s / kGramCS, nch * (s + 1) / kGramCS, sA, sB, acc);
    else gram_item<false>(A, m, J, ga.r, nullptr, ti, tj, nch * s / kGramCS, nch * (s + 1) / kGramCS, sA, sB, acc);
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) Pt[(16 * wr + 8 * i + gq) * 65 + 32 * wc + 8 * j + 2 * t + e] = acc[i][j][e];
    cluster.sync();
    const int64_t o0 = (int64_t)ti * GT, o1 = (int64_t)tj * GT;
    constexpr int RPR = GT / kGramCS;  // output rows reduced by each rank
    for (int e = tid; e < RPR * GT; e += 256) {  // columns fastest: contiguous DSMEM reads of the partial
      const int w = RPR * s + e / GT, k = e % GT;  // tiles (rows fastest coalesces the M stores but scatters
                                                   // the remote reads: r = 435 15.3 → 24.1 µs, measured)
      const int64_t oi = o0 + w, oj = o1 + k;
      if (oi < ga.nout && oj < ga.nout && oi >= oj) {
        double v = 0.0;
#pragma unroll
        for (int q = 0; q < kGramCS; ++q) v += cluster.map_shared_rank(Pt, q)[w * 65 + k];
        if (oi < ga.nmat) {
          double x = (ga.mult == 1.0 ? v : ga.mult * v) + (oi == oj ? ga.diag : 0.0);
          if (oi == oj && ga.jit != 0.0) x = __fma_rn(x, ga.jit, x);
          M[oi + oj * ga.ld] = x;
        } else {
          M[oi + oj * ga.ld] = v;  // rhs row (SMW: u = A_Jᵀ g)
        }
      }
    }
    cluster.sync();  // remote reads done before the next tile reuses the buffers
  }
}

// K3 split over the whole GPU (the hot-path Newton systems): k_gram_fused gives each 64 × 64 tile an
// 8-CTA cluster, and at m = 500 only 33 of the 36 m × m clusters fit at once (GPC packing), so a
// second round of 3 clusters doubled the time at large r.  Here the work items are (tile, K-slice)
// pairs with ns = min(grid / tiles, chunks / minch) slices per tile, so every item runs in ONE round of a
// cooperative launch (all CTAs co-resident): CTA b takes item b, sums its K-slice of the tile on
// the FP64 tensor cores (gram_item), stores the partial tile to P (L2, column-major), and arrives on the tile's
// counter; the ns CTAs of a tile wait for all ns partials, then slice s reduces rows
// [64s/ns, 64(s+1)/ns) of the tile over the slices in slice order (deterministic) with the
// k_gram_reduce epilogue (× mult, + diag, jitter, rhs row) straight into M.  The last CTA of a tile
// to finish resets its counters for the next launch.  Graph mode: branch and sizes from geo;
// only > 0 restricts to one branch (sharded SMW on gathered columns).
template <class Acc>
__global__ void __launch_bounds__(256, 2)
    k_gram_sk(const Acc A, int64_t m, const int32_t* __restrict__ J, double* __restrict__ M,
              const double* __restrict__ g, GramFusedArgs ga, const DirGeo* geo, int only, double* __restrict__ Pt,
              unsigned* __restrict__ cnt, int minch, const int64_t* __restrict__ r_loc = nullptr, int raw = 0) {
  __shared__ __align__(16) double sm[2 * kGramSmem];
  __shared__ bool last;
  if (geo) {
    if ((geo->branch != 1 && geo->branch != 2) || (only && geo->branch != only)) return;
    ga.branch = geo->branch;
    ga.r = geo->r;
    ga.nout = geo->nout;
    ga.nmat = geo->nmat;
    ga.tiles = geo->tiles;
    ga.ld = geo->ld;
    ga.diag = geo->diag;
    ga.mult = geo->mult;
    ga.jit = geo->jit;
  }
  if (raw) {  // §8(f3): the raw local partial Gram (m × m, ld = m) of a sharded rank's own columns
    if (r_loc) ga.r = *r_loc;
    ga.mult = 1.0;
    ga.diag = 0.0;
    ga.jit = 0.0;
    ga.ld = ga.nout;
    g = nullptr;
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, t = lane & 3, wr = warp >> 1, wc = warp & 1;
  const bool smw = ga.branch == 1;
  const int64_t K = smw ? m : ga.r;
  const int64_t nch = (K + 31) / 32;
  int ns = (int)gridDim.x / ga.tiles;  // slices per tile: one round, ≥ minch reduction chunks each (the
  if (ns > nch / minch) ns = (int)(nch / minch);  // partial tiles cost L2 traffic ∝ tiles · ns)
  if (ns < 1) ns = 1;
  if (!smw && g)  // the rhs row of Eq. (18): M[nmat + e·ld] = g[e]
    for (int64_t e = (int64_t)blockIdx.x * 256 + tid; e < ga.nmat; e += (int64_t)gridDim.x * 256)
      M[ga.nmat + e * ga.ld] = g[e];
  for (int item = blockIdx.x; item < ga.tiles * ns; item += gridDim.x) {  // one round when tiles ≤ grid
    const int tq = item / ns, s = item % ns;
    int ti, tj;
    tri_tile(tq, &ti, &tj);
    double acc[2][4][2];
    if (smw) gram_item<true>(A, m, J, ga.r, g, ti, tj, nch * s / ns, nch * (s + 1) / ns, sm, sm + kGramSmem, acc);
    else gram_item<false>(A, m, J, ga.r, nullptr, ti, tj, nch * s / ns, nch * (s + 1) / ns, sm, sm + kGramSmem, acc);
    double* Pi = Pt + (size_t)item * GT * GT;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) __stcg(Pi + (32 * wc + 8 * j + 2 * t + e) * GT + 16 * wr + 8 * i + gq, acc[i][j][e]);
    __threadfence();
    __syncthreads();
    if (tid == 0) {
      atomicAdd(cnt + 2 * tq, 1u);
      while (atomicAdd(cnt + 2 * tq, 0u) < (unsigned)ns) {
      }
      __threadfence();
    }
    __syncthreads();
    const int64_t o0 = (int64_t)ti * GT, o1 = (int64_t)tj * GT;
    const int w0 = GT * s / ns, w1 = GT * (s + 1) / ns;
    const double* Pb = Pt + (size_t)tq * ns * GT * GT;
    const int nr = w1 - w0;
    for (int e = tid; e < nr * GT; e += 256) {  // rows fastest: contiguous partial-tile columns and M segments
      const int w = w0 + e % nr, k = e / nr;
      const int64_t oi = o0 + w, oj = o1 + k;
      if (oi < ga.nout && oj < ga.nout && oi >= oj) {
        double v = 0.0;
        for (int q = 0; q < ns; ++q) v += __ldcg(Pb + (size_t)q * GT * GT + k * GT + w);
        if (oi < ga.nmat) {
          double x = (ga.mult == 1.0 ? v : ga.mult * v) + (oi == oj ? ga.diag : 0.0);
          if (oi == oj && ga.jit != 0.0) x = __fma_rn(x, ga.jit, x);
          M[oi + oj * ga.ld] = x;
        } else {
          M[oi + oj * ga.ld] = v;  // rhs row (SMW: u = A_Jᵀ g)
        }
      }
    }
    __syncthreads();
    if (tid == 0) {  // the tile's last finisher resets both counters (every waiter is past its wait)
      last = atomicAdd(cnt + 2 * tq + 1, 1u) == (unsigned)ns - 1;
      if (last) {
        cnt[2 * tq] = 0u;
        cnt[2 * tq + 1] = 0u;
      }
    }
    __syncthreads();
  }
}

template <bool SMW, class Acc>
__global__ void __launch_bounds__(256) k_gram(const Acc A, int64_t m, const int32_t* __restrict__ J, int64_t r,
                                              double* __restrict__ W, const double* __restrict__ gext, int tiles,
                                              int ns, const DirGeo* geo) {
  __shared__ double sA[kGramSmem], sB[kGramSmem];
  if (geo) {
    if (geo->branch != (SMW ? 1 : 2)) return;
    r = geo->r;
    tiles = geo->tiles;
    ns = geo->ns;
  }
  gram_body<SMW>(A, m, J, r, W, gext, tiles, ns, sA, sB);
}

// Warp loads rows [r0, r0+32) × cols [c0, c0+32) of M into S (row-major, TLD), zero outside
// rows < nr and cols < nc.  One 256-B coalesced load per column (lane = row).
SSN_DEV void load_tile_rows(const double* M, int ld, int r0, int c0, int nr, int nc, double* S, int lane) {
  const bool rok = r0 + lane < nr;
  const double* col = M + (int64_t)c0 * ld + (rok ? r0 + lane : 0);
  const int ncl = nc - c0;
  double v[CHT];  // all 32 loads in flight before the smem stores
#pragma unroll
  for (int p = 0; p < CHT; ++p) v[p] = (rok && p < ncl) ? __ldcg(col + p * ld) : 0.0;
#pragma unroll
  for (int p = 0; p < CHT; ++p) S[lane * TLD + p] = v[p];
}

// The diagonal team (CTA 0 warps 0-3, t128 ∈ [0,128), named barrier 2) factors the diagonal tile
// S (smem, row-major: S[r][c] = A[n0+r][n0+c]) and inverts the factor, blocked by 8 columns.
// Warp w owns columns [8w, 8w+8) of every row (lane = row: a[q] = L[lane][8w+q]), a replica of
// their diagonal entries (dgw, updated with the same fma as the owning lane — bitwise equal), and
// rows [8w, 8w+8) of W = L⁻¹ (lane = column: wr[q] = W[8w+q][lane]).
//   block b = 0..3: warp b factors its 8 columns with intra-warp shuffles (per pivot j: rsqrt →
//   scale column → shuffle → rank-1 update of its later columns; W row j /= L_jj, later rows
//   −= L_kj · row j — column-oriented forward substitution on I), publishes the 8 columns of L
//   and 8 rows of W to smem (double-buffered), one 128-thread barrier.  The next owner (b + 1)
//   applies block b's rank-8 update lazily, one column right before its pivot (off the chain);
//   warps > b + 1 apply it eagerly while the next block is factored.
// Rows ≥ kn (appended rows / padding) are identity-padded and never pivot.  Writes L (rows <
// nrow, cols < kn, c ≤ r) into M at (n0, n0), W (row-major 32 × 32) to Wout and to Wsm (smem,
// row stride TLD).  Compact code (block loop rolled): it runs once per panel.
// smem scratch `cb`: 2 × (32 × 9 + 8 × 33) doubles.
constexpr int kDiagScratch = 2 * (CHT * 9 + 8 * 33);
SSN_DEV void diag_factor4(const double* S, double* M, int ld, int n0, int kn, int nrow, double* Wout, double* Wsm,
                          int* info, double* cb, int t128) {
  const int w = t128 >> 5, lane = t128 & 31;
  double a[8], dgw[8], wr[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int c = 8 * w + q;
    a[q] = (lane < nrow && c < kn) ? S[lane * TLD + c] : (lane == c ? 1.0 : 0.0);
    dgw[q] = (c < kn) ? S[c * TLD + c] : 1.0;
    wr[q] = (lane == c) ? 1.0 : 0.0;
  }
  bool bad = false;
#pragma unroll 1
  for (int blk = 0; blk < 4; ++blk) {
    double* Lb = cb + (blk & 1) * (CHT * 9 + 8 * 33);  // Lb[r * 9 + p] = L[r][8blk + p]
    double* Wb = Lb + CHT * 9;                          // Wb[p * 33 + c] = W[8blk + p][c]
    if (w == blk) {
      const double* Lp = cb + ((blk + 1) & 1) * (CHT * 9 + 8 * 33);  // block blk − 1
      const double* Wp = Lp + CHT * 9;
      double lrp[8], wbp[8];
      if (blk > 0) {
#pragma unroll
        for (int pp = 0; pp < 8; ++pp) {
          lrp[pp] = Lp[lane * 9 + pp];
          wbp[pp] = Wp[pp * 33 + lane];
        }
      }
      if (blk > 0) {  // rank-8 update of this block's columns from block blk − 1, before any pivot:
                      // eight independent chains, so only pivot 0 waits for one of them
#pragma unroll
        for (int p = 0; p < 8; ++p)
#pragma unroll
          for (int pp = 0; pp < 8; ++pp) {
            const double l = Lp[(8 * w + p) * 9 + pp];
            dgw[p] = fma(-l, l, dgw[p]);
            a[p] = fma(-lrp[pp], l, a[p]);
            wr[p] = fma(-l, wbp[pp], wr[p]);
          }
      }
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int j = 8 * blk + p;
        double d = dgw[p];
        bad |= (j < kn) && !(d > 0.0);
        d = (j < kn && d > 0.0) ? d : 1.0;
        const double inv = rsqrt_pos(d);
        const double lij = (lane > j) ? a[p] * inv : (lane == j ? d * inv : 0.0);
        const double wj = wr[p] * inv;  // W row j scaled (final)
#pragma unroll
        for (int q = p + 1; q < 8; ++q) {
          const double lq = __shfl_sync(0xffffffffu, lij, 8 * blk + q);  // L[8blk+q][j]
          dgw[q] = fma(-lq, lq, dgw[q]);
          a[q] = fma(-lij, lq, a[q]);
          wr[q] = fma(-lq, wj, wr[q]);
        }
        a[p] = lij;
        wr[p] = wj;
      }
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        Lb[lane * 9 + p] = a[p];
        Wb[p * 33 + lane] = wr[p];
      }
    }
    asm volatile("bar.sync 2, 128;" ::: "memory");
    if (w > blk + 1) {  // eager rank-8 update from block blk
      double lr[8], wb[8];
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        lr[p] = Lb[lane * 9 + p];
        wb[p] = Wb[p * 33 + lane];
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const double* lc = Lb + (8 * w + q) * 9;
#pragma unroll
        for (int p = 0; p < 8; ++p) {
          const double l = lc[p];  // L[8w+q][8blk+p]
          dgw[q] = fma(-l, l, dgw[q]);
          a[q] = fma(-lr[p], l, a[q]);
          wr[q] = fma(-l, wb[p], wr[q]);
        }
      }
    }
  }
  if (bad && lane == 0) atomicExch(info, 1);
  if (!M) asm volatile("bar.sync 2, 128;" ::: "memory");  // every warp has read S before L overwrites it
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int c = 8 * w + q;
    if (M) {
      if (lane < nrow && c < kn && c <= lane) M[(int64_t)(n0 + lane) + (int64_t)(n0 + c) * ld] = a[q];
    } else {  // L into the smem tile itself (DSMEM-resident factor): rows < nrow, cols < kn, else 0
      const_cast<double*>(S)[lane * TLD + c] = (lane < nrow && c < kn && c <= lane) ? a[q] : 0.0;
    }
    const double wv = (c < kn && lane < kn) ? wr[q] : (lane == c ? 1.0 : 0.0);  // pad: identity
    if (Wout) Wout[c * CHT + lane] = wv;
    if (Wsm) Wsm[c * TLD + lane] = wv;
  }
}

// Backward substitution v = L⁻ᵀ z by one CTA (8 warps), right-looking over 32-blocks:
//   for b = last … 0:  v_b = W_bᵀ z_b  (warp 0)  |  z_a −= L_baᵀ v_b for a < b (warp a mod 8)
// z (smem, N) holds the forward-substitution result on entry and v on exit.  W blocks are staged
// in a smem ring (≤ 16 blocks).  Each warp prefetches its first L tile of the next step into
// registers (coalesced: lane = row) while the current step runs and transposes it through its
// own smem tile (lane = column for the dot products); further tiles (N > 256) load on demand.
constexpr int kBwdRing = 16;
SSN_DEV void bwd_tile_load(const double* M, int ld, int N, int b, int a, double (&t)[CHT], int lane) {
  const int row = b * CHT + lane;
  const bool rok = row < N;
  const double* src = M + (int64_t)a * CHT * ld + (rok ? row : 0);
#pragma unroll
  for (int c = 0; c < CHT; ++c) t[c] = rok ? __ldcg(src + c * ld) : 0.0;
}
SSN_DEV void backward_solve(const double* M, int ld, int N, const double* Winv, double* z, double* Wring, double* Tw,
                            int tid) {
  const int warp = tid >> 5, lane = tid & 31;
  const int ntc = (N + CHT - 1) / CHT;
  double* Ts = Tw + (size_t)warp * CHT * TLD;  // this warp's transpose tile
  auto stage_w = [&](int b) {  // W_b → ring slot b % kBwdRing (all threads)
    double* dst = Wring + (size_t)(b % kBwdRing) * CHT * CHT;
    const double* src = Winv + (size_t)b * CHT * CHT;
    for (int e = tid; e < CHT * CHT; e += blockDim.x) dst[e] = __ldcg(src + e);
  };
  for (int b = ntc - 1; b >= 0 && b >= ntc - kBwdRing; --b) stage_w(b);
  double cur[CHT], nxt[CHT];  // tile (b, warp): cur[c] = L[b0 + lane][a0 + c]
  if (warp < ntc - 1) bwd_tile_load(M, ld, N, ntc - 1, warp, cur, lane);
  __syncthreads();
  // z_a −= L_baᵀ v_b for one tile held as t[c] = L[b0 + lane][a0 + c] (zero rows ≥ N)
  auto upd = [&](int a, int b0, const double (&t)[CHT]) {
#pragma unroll
    for (int c = 0; c < CHT; ++c) Ts[lane * TLD + c] = t[c];
    __syncwarp();
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
    for (int r = 0; r < CHT; r += 4) {  // lane = column: Σ_r L[b0+r][a0+lane] v[b0+r]
      s0 = fma(Ts[r * TLD + lane], z[b0 + r], s0);
      s1 = fma(Ts[(r + 1) * TLD + lane], z[b0 + r + 1], s1);
      s2 = fma(Ts[(r + 2) * TLD + lane], z[b0 + r + 2], s2);
      s3 = fma(Ts[(r + 3) * TLD + lane], z[b0 + r + 3], s3);
    }
    z[a * CHT + lane] -= (s0 + s1) + (s2 + s3);  // a < b: full block
    __syncwarp();
  };
#pragma unroll 1
  for (int b = ntc - 1; b >= 0; --b) {
    const int b0 = b * CHT, bn = min(CHT, N - b0);
    if (warp < b - 1) bwd_tile_load(M, ld, N, b - 1, warp, nxt, lane);  // prefetch
    if (warp == 0) {  // v_b[c] = Σ_r W_b[r][c] z_b[r]   (W_b lower triangular)
      const double* Wb = Wring + (size_t)(b % kBwdRing) * CHT * CHT;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
      for (int r = 0; r < CHT; r += 4) {
        const double z0 = (r < bn) ? z[b0 + r] : 0.0, z1 = (r + 1 < bn) ? z[b0 + r + 1] : 0.0;
        const double z2 = (r + 2 < bn) ? z[b0 + r + 2] : 0.0, z3 = (r + 3 < bn) ? z[b0 + r + 3] : 0.0;
        s0 = fma(Wb[r * CHT + lane], z0, s0);
        s1 = fma(Wb[(r + 1) * CHT + lane], z1, s1);
        s2 = fma(Wb[(r + 2) * CHT + lane], z2, s2);
        s3 = fma(Wb[(r + 3) * CHT + lane], z3, s3);
      }
      __syncwarp();
      z[b0 + lane] = (lane < bn) ? (s0 + s1) + (s2 + s3) : 0.0;  // zero pad beyond N (z has 1024 slots)
    }
    __syncthreads();
    if (b - kBwdRing >= 0) stage_w(b - kBwdRing);  // ring slot of b is free now
    if (warp < b) upd(warp, b0, cur);
#pragma unroll 1
    for (int a = warp + 8; a < b; a += 8) {  // further tiles of this warp: on demand
      double t[CHT];
      bwd_tile_load(M, ld, N, b, a, t, lane);
      upd(a, b0, t);
    }
#pragma unroll
    for (int c = 0; c < CHT; ++c) cur[c] = nxt[c];
    __syncthreads();
  }
}

// dynamic shared memory of k_chol_cluster (bytes): factorisation operands, or in the backward
// solve z (1024) + the W ring
constexpr int kQuadTiles = 7 + kColSlots;  // per quad: 2 stages × (L_ik, L_jk, A_ij), W_{k+1}, slots
constexpr size_t kCholSmemFact =
    (size_t)(2 * kQuadTiles * CHT * TLD + 2 * CHT * TLD + kDiagScratch) * sizeof(double);
constexpr size_t kCholSmemBwd = (size_t)(1024 + kBwdRing * CHT * CHT + 8 * CHT * TLD) * sizeof(double);
constexpr size_t kCholSmem = kCholSmemFact > kCholSmemBwd ? kCholSmemFact : kCholSmemBwd;

// NR ≥ N + 1 rows: rows N..NR-1 are appended rows C, which leave the factorisation as C L⁻ᵀ.
// With out != nullptr row N is the right-hand side and the backward solve runs; otherwise the
// kernel stops after the factorisation (e.g. degrees of freedom from C = A_J).
__global__ void __launch_bounds__(256, 1) k_chol_cluster(double* M, int N, int NR, int ld, double* __restrict__ out,
                                                         double scale, const double* __restrict__ dotv,
                                                         double* dot_out, double* Winv, int* info,
                                                         const double* __restrict__ ybase, double* __restrict__ yt,
                                                         const DirGeo* geo, int want, int* kflag, int nmin,
                                                         const CholArgs* ca) {
  namespace cg = cooperative_groups;
  if (geo) {  // graph mode: order from the device geometry; whole cluster exits together
    if ((want >= 0 ? geo->branch != want : (geo->branch != 1 && geo->branch != 2)) || geo->N < nmin) return;
    if (ca) {
      const CholArgs& c = ca[geo->branch - 1];
      out = c.out;
      scale = c.scale;
      dotv = c.dotv;
      dot_out = c.dot_out;
      ybase = c.ybase;
      yt = c.yt;
    }
    N = geo->N;
    NR = geo->NR;
    ld = geo->ld;
  }
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank(), CS = (int)cl.num_blocks();
  extern __shared__ double dsm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quad = warp >> 2, qw = warp & 3;
  const int g = lane >> 2, t = lane & 3;
  // smem: per quad [SA, SB, Wq, slots × kColSlots] (tiles 32 × TLD); CTA 0 adds T2, T3, scratch
  double* QB = dsm + (size_t)quad * kQuadTiles * CHT * TLD;
  double* SA = QB;                       // stage s: QB + 3s tiles = L_ik, + 1 = L_jk, + 2 = A_ij
  double* Wq = QB + 6 * CHT * TLD;       // W_{k+1} for this quad's TRSMs
  double* slots = QB + 7 * CHT * TLD;    // updated column-(k+1) tiles awaiting W_{k+1}
  double* T2 = dsm + (size_t)2 * kQuadTiles * CHT * TLD;  // CTA-0 diagonal tile
  double* T3 = T2 + CHT * TLD;                                  // CTA-0: L_{k+1,k}
  double* dscr = T3 + CHT * TLD;                                // diag_factor4 scratch
  const int ntc = (N + CHT - 1) / CHT, ntr = (NR + CHT - 1) / CHT;
  // Roles.  CTA 0 quad 0 = the diagonal team (the critical chain).  Worker quads: every quad of
  // the other CTAs (CTA 0 quad 1 too when the cluster has one CTA).
  const bool diag_team = (rank == 0 && quad == 0);
  const int NQ = (CS > 1) ? 2 * (CS - 1) : 1;
  const int gq = (CS > 1) ? ((rank == 0) ? -1 : 2 * (rank - 1) + quad) : (quad == 1 ? 0 : -1);
  const int qbar = 3 + quad;  // named barrier of this quad (128 threads)
#ifdef CHOL_PROBE
#define STAMP(i) do { if (rank == 0 && tid == 0 && (i) < 64) { unsigned long long t_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); g_t[i] = t_; g_c[i] = clock64(); } } while (0)
#define STAMPW(i) do { if (rank == 1 && tid == 0 && (i) < 64) { unsigned long long t_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); g_t[i] = t_; g_c[i] = clock64(); } } while (0)
#else
#define STAMP(i) do {} while (0)
#define STAMPW(i) do {} while (0)
#endif
  STAMP(0);
  if (rank == 0 && tid < ntc + 1) kflag[tid] = 0;  // W-ready flags of this launch
  cl.sync();
  // One phase per panel.  M(k), k = −1 … ntc−2:
  //   diagonal team: A_{k+1,k+1} −= L_{k+1,k} L_{k+1,k}ᵀ (k ≥ 0), factor it → L, W_{k+1}; publish
  //                  W_{k+1} (global) with a release flag
  //   worker quads:  column-(k+1) tiles (i ≥ k+2): A_{i,k+1} −= L_ik L_{k+1,k}ᵀ into a smem slot;
  //                  trailing tiles (i, j ≥ k+2): A_ij −= L_ik L_jkᵀ in place;
  //                  then wait for W_{k+1} (acquire) and TRSM the slots: L_{i,k+1} = A_{i,k+1} W_{k+1}ᵀ
  //   cluster barrier (column k+1 of L complete in M)
  for (int k = -1; k + 1 < ntc; ++k) {
    const int k0 = k * CHT, kn = (k >= 0) ? min(CHT, N - k0) : 0;
    const int c0 = (k + 1) * CHT, cn = min(CHT, N - c0);  // the column being factored / TRSM'd
    if (diag_team) {
      if (k < 0) {
        if (warp == 0) load_tile_rows(M, ld, 0, 0, NR, N, T2, lane);
      } else {
        // L_{k+1,k} (rows c0.., panel k) and A_{k+1,k+1}, then the DMMA update (8 rows per warp)
        {  // coalesced: lane = row, warp qw takes columns 8qw .. 8qw+7
          const bool rok = c0 + lane < NR;
          const double* src = M + (int64_t)(k0 + 8 * qw) * ld + (rok ? c0 + lane : 0);
          double v[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] = (rok && 8 * qw + e < kn) ? __ldcg(src + e * ld) : 0.0;
#pragma unroll
          for (int e = 0; e < 8; ++e) T3[lane * TLD + 8 * qw + e] = v[e];
        }
        double acc[4][2];
        const int r = c0 + 8 * qw + g;
#pragma unroll
        for (int cb = 0; cb < 4; ++cb)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int c = c0 + 8 * cb + 2 * t + e;
            acc[cb][e] = (r < NR && c < N) ? __ldcg(M + (int64_t)r + (int64_t)c * ld) : 0.0;
          }
        asm volatile("bar.sync 2, 128;" ::: "memory");
        strip_mma(T3, T3, acc, -1.0, qw, lane);
#pragma unroll
        for (int cb = 0; cb < 4; ++cb)
#pragma unroll
          for (int e = 0; e < 2; ++e) T2[(8 * qw + g) * TLD + 8 * cb + 2 * t + e] = acc[cb][e];
      }
      asm volatile("bar.sync 2, 128;" ::: "memory");
      if (k == 1) STAMP(48);
#if defined(CHOL_EXPERIMENT) && CHOL_EXPERIMENT == 3
      if (false)
#endif
      diag_factor4(T2, M, ld, c0, cn, min(CHT, NR - c0), Winv + (size_t)(k + 1) * CHT * CHT, nullptr, info, dscr,
                   tid);
      __threadfence();                                 // this thread's W_{k+1} / L stores, gpu scope
      asm volatile("bar.sync 2, 128;" ::: "memory");  // … for all 128 threads before the release
      if (tid == 0) {
        __threadfence();
        asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(kflag + k + 1), "r"(1) : "memory");
      }
      if (k == 1) STAMP(49);
    } else if (gq >= 0) {
      const int ncol = ntr - k - 2;                       // column-(k+1) tiles i = k+2 …
      const int remc = ntc - k - 2, remr = ntr - k - 2;   // trailing: columns k+2 … ntc−1
      const int ntri = remc > 0 ? remc * (remc + 1) / 2 : 0;
      const int ntrail = (k >= 0 && remc > 0) ? ntri + (remr - remc) * remc : 0;
      int nslot = 0;
      // job q → tile (i0, j0); column jobs (q < ncol) first.  The three operand tiles of job q + NQ
      // stream global → smem with cp.async (no register staging) while job q computes; two stages.
      auto job_tile = [&](int q, int& i0, int& j0) {
        if (q < ncol) {
          i0 = (k + 2 + q) * CHT;
          j0 = c0;
        } else {
          const int e = q - ncol;
          int ii, jj;
          if (e < ntri) tri_tile(e, &ii, &jj);
          else {
            const int f = e - ntri;
            ii = remc + f / remc;
            jj = f % remc;
          }
          i0 = (k + 2 + ii) * CHT;
          j0 = (k + 2 + jj) * CHT;
        }
      };
      const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(SA);
      auto cp8 = [&](double* dst, const double* src, bool ok) {  // 8-byte async copy or a zero
        if (ok) {
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                       "l"(src)
                       : "memory");
        } else {
          *dst = 0.0;
        }
      };
      (void)sbase;
      // issue: lane = row, warp qw takes columns 8qw .. 8qw+7 of the three tiles
      auto issue = [&](int q, int st) {
        int i0, j0;
        job_tile(q, i0, j0);
        double* tA = SA + (size_t)(3 * st) * CHT * TLD;
        double* tB = tA + CHT * TLD;
        double* tC = tB + CHT * TLD;
        const bool ra = i0 + lane < NR, rb = j0 + lane < N;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int c = 8 * qw + e;
          cp8(tC + lane * TLD + c, M + (int64_t)(j0 + c) * ld + i0 + lane, ra && j0 + c < N);
          if (k >= 0) {
            cp8(tA + lane * TLD + c, M + (int64_t)(k0 + c) * ld + i0 + lane, ra && c < kn);
            cp8(tB + lane * TLD + c, M + (int64_t)(k0 + c) * ld + j0 + lane, rb && c < kn);
          }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      };
      const int njobs = ncol + ntrail;
      if (gq < njobs) issue(gq, 0);
      if (k == 1) STAMPW(50);
      int st = 0;
#pragma unroll 1
      for (int q = gq; q < njobs; q += NQ, st ^= 1) {
        int i0, j0;
        job_tile(q, i0, j0);
        const bool colj = q < ncol;
        if (q + NQ < njobs) {
          issue(q + NQ, st ^ 1);
          asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
          asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        asm volatile("bar.sync %0, 128;" ::"r"(qbar) : "memory");
        if (k == 1 && q == gq) STAMPW(51);
        const double* tA = SA + (size_t)(3 * st) * CHT * TLD;
        const double* tB = tA + CHT * TLD;
        const double* tC = tB + CHT * TLD;
        double cur[4][2];
#pragma unroll
        for (int cb = 0; cb < 4; ++cb)
#pragma unroll
          for (int e = 0; e < 2; ++e) cur[cb][e] = tC[(8 * qw + g) * TLD + 8 * cb + 2 * t + e];
#if defined(CHOL_EXPERIMENT) && CHOL_EXPERIMENT == 1
        if (false)
#endif
        if (k >= 0) strip_mma(tA, tB, cur, -1.0, qw, lane);
        if (k == 1 && q == gq) STAMPW(53);
        // column tiles beyond the slots (small clusters, many appended rows) go back to M in place
        double* dst = (colj && nslot < kColSlots) ? slots + (size_t)nslot * CHT * TLD : nullptr;
        if (colj) ++nslot;
        const int r = i0 + 8 * qw + g;
        if (dst) {  // keep for the TRSM (full tile, zero outside)
#pragma unroll
          for (int cb = 0; cb < 4; ++cb)
#pragma unroll
            for (int e = 0; e < 2; ++e) dst[(8 * qw + g) * TLD + 8 * cb + 2 * t + e] = cur[cb][e];
        } else {
#pragma unroll
          for (int cb = 0; cb < 4; ++cb)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int rl = 8 * qw + g, cl_ = 8 * cb + 2 * t + e;
              const int c = j0 + cl_;
              if (r < NR && c < N && (i0 != j0 || cl_ <= rl)) M[(int64_t)r + (int64_t)c * ld] = cur[cb][e];
            }
        }
        asm volatile("bar.sync %0, 128;" ::"r"(qbar) : "memory");  // stage reuse
        if (k == 1 && q == gq) STAMPW(54);
        if (k == 1 && q == gq + NQ) STAMPW(55);
      }
      if (k == 1) STAMPW(56);
      if (nslot > 0) {  // TRSM of this quad's column tiles with W_{k+1}
        if (tid % 128 == 0) {
          int f;
          do {
            asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(f) : "l"(kflag + k + 1) : "memory");
            if (!f) __nanosleep(64);
          } while (!f);
        }
        asm volatile("bar.sync %0, 128;" ::"r"(qbar) : "memory");
        if (k == 1) STAMPW(57);
        {
          const double* Wk = Winv + (size_t)(k + 1) * CHT * CHT;
          const int tq = tid & 127;
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = __ldcg(Wk + tq + 128 * u);
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int e = tq + 128 * u;
            Wq[(e >> 5) * TLD + (e & 31)] = v[u];
          }
        }
        asm volatile("bar.sync %0, 128;" ::"r"(qbar) : "memory");
        int s = 0;
#pragma unroll 1
        for (int q = gq; q < ncol; q += NQ, ++s) {
          const int r0 = (k + 2 + q) * CHT;
          const double* src = slots + (size_t)s * CHT * TLD;
          if (s >= kColSlots) {  // overflow tile: reload the updated A_{i,k+1} from M into SA
            const bool rok = r0 + lane < NR;
            const double* sp = M + (int64_t)(c0 + 8 * qw) * ld + (rok ? r0 + lane : 0);
            double v[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] = (rok && 8 * qw + e < cn) ? __ldcg(sp + e * ld) : 0.0;
            asm volatile("bar.sync %0, 128;" ::"r"(qbar) : "memory");  // previous SA readers done
#pragma unroll
            for (int e = 0; e < 8; ++e) SA[lane * TLD + 8 * qw + e] = v[e];
            asm volatile("bar.sync %0, 128;" ::"r"(qbar) : "memory");
            src = SA;
          }
          double acc[4][2];
#pragma unroll
          for (int cb = 0; cb < 4; ++cb) acc[cb][0] = acc[cb][1] = 0.0;
          strip_mma(src, Wq, acc, 1.0, qw, lane);
          const int r = r0 + 8 * qw + g;
#pragma unroll
          for (int cb = 0; cb < 4; ++cb)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int c = 8 * cb + 2 * t + e;
              if (r < NR && c < cn) M[(int64_t)r + (int64_t)(c0 + c) * ld] = acc[cb][e];
            }
        }
      }
    }
    if (k == 1) STAMPW(58);
    cl.sync();
    STAMP(2 + k);
  }
  STAMP(40);
  if (out == nullptr) return;
  // ---- backward substitution v = L⁻ᵀ z (z = row N) ----
  // Cluster version when every CTA can stage its share in smem: CTA c owns the column blocks
  // a ≡ c (mod CS) and holds z_a, W_a and the tiles L_ba (b > a).  Step b (descending): the owner of
  // block b computes v_b = W_bᵀ z_b and writes it into every CTA's v buffer (DSMEM) | cluster barrier
  // | every CTA applies z_a −= L_baᵀ v_b to its blocks a < b.  Otherwise CTA 0 alone (backward_solve).
  int own_tiles = 0;  // rank 0 owns the most: blocks 0, CS, 2CS, …
  for (int a = 0; a < ntc; a += CS) own_tiles += ntc - a;  // tiles below + W_a
  const int kBwdTileBudget = (int)((kCholSmem / sizeof(double) - 1024 - 64 * CHT) / (CHT * TLD));
  if (CS > 1 && own_tiles <= kBwdTileBudget) {
    double* vfull = dsm;                        // 1024: v, filled block by block (broadcast)
    double* zl = dsm + 1024;                    // 64 × 32: z of the owned blocks (≤ 64 blocks)
    double* tl = zl + 64 * CHT;                 // staged tiles (TLD layout)
    // staging: for owned block a: W_a, then L_ba for b = a+1 … ntc−1, as one flat list of tiles
    // (8 independent loads in flight per thread)
    int nt = 0;
    for (int a = rank; a < ntc; a += CS) {
      const int a0 = a * CHT, an = min(CHT, N - a0);
      for (int e = tid; e < CHT; e += blockDim.x) zl[(a / CS) * CHT + e] = (e < an) ? __ldcg(M + (int64_t)N + (int64_t)(a0 + e) * ld) : 0.0;
      nt += ntc - a;
    }
    {
      const int total = nt * CHT * CHT;
      for (int base = tid; base < total; base += 8 * (int)blockDim.x) {
        double v[8];
        int dsti[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int idx = base + u * (int)blockDim.x;
          v[u] = 0.0;
          dsti[u] = -1;
          if (idx < total) {
            int tt = idx >> 10, e = idx & 1023;
            // tile tt → (a, b): walk the owned blocks
            int a = rank;
            while (tt >= ntc - a) {
              tt -= ntc - a;
              a += CS;
            }
            const int b = a + tt;  // tt = 0 → W_a
            const int r = e & 31, c = e >> 5;
            const int ti = idx >> 10;
            if (b == a) {
              v[u] = __ldcg(Winv + (size_t)a * CHT * CHT + (size_t)c * CHT + r);  // W_a[c][r]
              dsti[u] = ti * CHT * TLD + c * TLD + r;
            } else {
              const int row = b * CHT + r;
              v[u] = (row < N) ? __ldcg(M + (int64_t)row + (int64_t)(a * CHT + c) * ld) : 0.0;
              dsti[u] = ti * CHT * TLD + r * TLD + c;
            }
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (dsti[u] >= 0) tl[dsti[u]] = v[u];
      }
    }
    __syncthreads();
    STAMP(41);
    // tile index of (b, a) for owned a: block offset of a + 1 + (b − a − 1)
    auto tile_of = [&](int a, int b) {
      int off = 0;
      for (int a2 = rank; a2 < a; a2 += CS) off += ntc - a2;
      return tl + (size_t)(off + (b - a)) * CHT * TLD;  // b == a → W_a
    };
    for (int b = ntc - 1; b >= 0; --b) {
      const int b0 = b * CHT, bn = min(CHT, N - b0);
      if (b % CS == rank && warp == 0) {  // v_b = W_bᵀ z_b, broadcast to every CTA
        const double* Wt = tile_of(b, b);
        const double* zb = zl + (b / CS) * CHT;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
        for (int r = 0; r < CHT; r += 4) {
          s0 = fma(Wt[r * TLD + lane], zb[r], s0);
          s1 = fma(Wt[(r + 1) * TLD + lane], zb[r + 1], s1);
          s2 = fma(Wt[(r + 2) * TLD + lane], zb[r + 2], s2);
          s3 = fma(Wt[(r + 3) * TLD + lane], zb[r + 3], s3);
        }
        const double v = (lane < bn) ? (s0 + s1) + (s2 + s3) : 0.0;
        for (int q = 0; q < CS; ++q) cl.map_shared_rank(vfull, q)[b0 + lane] = v;
      }
      cl.sync();
      // z_a −= L_baᵀ v_b for owned a < b (one warp per owned block)
      int ia = 0;
      for (int a = rank; a < b; a += CS, ++ia) {
        if (warp != ia) continue;
        const double* Tt = tile_of(a, b);
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
        for (int r = 0; r < CHT; r += 4) {
          s0 = fma(Tt[r * TLD + lane], vfull[b0 + r], s0);
          s1 = fma(Tt[(r + 1) * TLD + lane], vfull[b0 + r + 1], s1);
          s2 = fma(Tt[(r + 2) * TLD + lane], vfull[b0 + r + 2], s2);
          s3 = fma(Tt[(r + 3) * TLD + lane], vfull[b0 + r + 3], s3);
        }
        zl[(a / CS) * CHT + lane] -= (s0 + s1) + (s2 + s3);
      }
      __syncthreads();
    }
    STAMP(42);
    if (rank != 0) return;
    double* zv = vfull;
    __shared__ double redc[8];
    double dot = 0.0;
    for (int i = tid; i < N; i += blockDim.x) {
      const double v = scale * zv[i];
      out[i] = v;
      if (yt) yt[i] = __dadd_rn(ybase[i], __dmul_rn(1.0, v));  // Armijo trial y + d (m × m branch)
      if (dotv) dot += dotv[i] * v;
    }
    if (dotv) {
      dot = warp_allsum(dot);
      if (lane == 0) redc[warp] = dot;
      __syncthreads();
      if (tid == 0) {
        double sacc = 0.0;
        for (int wi = 0; wi < 8; ++wi) sacc += redc[wi];
        *dot_out = sacc;
      }
    }
    return;
  }
  if (rank != 0) return;
  double* zv = dsm;                          // N doubles (N ≤ 1024)
  double* Wring = dsm + 1024;                // kBwdRing × 32 × 32 doubles
  double* Tw = Wring + kBwdRing * CHT * CHT;  // 8 warps × 32 × TLD transpose tiles
  for (int i = tid; i < N; i += blockDim.x) zv[i] = __ldcg(M + (int64_t)N + (int64_t)i * ld);
  __syncthreads();
  STAMP(41);
  backward_solve(M, ld, N, Winv, zv, Wring, Tw, tid);
  STAMP(42);
  __shared__ double red[8];
  double dot = 0.0;
  for (int i = tid; i < N; i += blockDim.x) {
    const double v = scale * zv[i];
    out[i] = v;
    if (yt) yt[i] = __dadd_rn(ybase[i], __dmul_rn(1.0, v));  // Armijo trial y + d (m × m branch)
    if (dotv) dot += dotv[i] * v;
  }
  if (dotv) {
    dot = warp_allsum(dot);
    if (lane == 0) red[warp] = dot;
    __syncthreads();
    if (tid == 0) {
      double sacc = 0.0;
      for (int wi = 0; wi < 8; ++wi) sacc += red[wi];
      *dot_out = sacc;
    }
  }
}


// y ← y + s·d  (m-vector) and small helpers
__global__ void k_axpy_m(int64_t m, const double* y, double s, const double* d, double* out, const double* sp) {
  if (sp) s = *sp;
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < m) out[k] = __dadd_rn(y[k], __dmul_rn(s, d[k]));
}
__global__ void k_neg_copy(int64_t m, const double* g, double* d, const double* dotv, double* dot_out,
                           const double* y, double* yt, const DirGeo* geo) {
  __shared__ double red[32];
  if (geo && geo->branch != 0) return;
  double dot = 0.0;
  for (int64_t k = threadIdx.x; k < m; k += blockDim.x) {
    d[k] = -g[k];
    if (yt) yt[k] = __dadd_rn(y[k], __dmul_rn(1.0, -g[k]));
    dot += dotv[k] * (-g[k]);
  }
  dot = warp_allsum(dot);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = dot;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int wi = 0; wi < (int)(blockDim.x >> 5); ++wi) s += red[wi];
    *dot_out = s;
  }
}

// x ← P: zero x on the old support, then scatter (J, P_J).
__global__ void k_zero_at(const int32_t* __restrict__ idx, int64_t cnt, const int64_t* cnt_dev, double* x,
                          const int* skip) {
  if (skip && *skip) return;
  if (cnt < 0) cnt = *cnt_dev;  // grid-stride with a device-resident count
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x)
    x[idx[i]] = 0.0;
}

// y = (*r_dev > 0) ? −b + Σ_{valid b'} parts[b'] : 0    (warm start y0 = A x0 − b, reading R8)
__global__ void k_init_y(int64_t m, const double* __restrict__ bvec, const double* __restrict__ parts,
                         const int* __restrict__ valid, int nparts, const int64_t* r_dev, double* __restrict__ y) {
  const bool warm = *r_dev > 0;
  for (int64_t k = threadIdx.x; k < m; k += blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nparts; ++b)
      if (!valid || valid[b]) s += parts[(size_t)b * m + k];
    y[k] = warm ? (-1.0 * bvec[k] + s) : 0.0;
  }
}
__global__ void k_to_i64(const double* src, int64_t* dst) { *dst = (int64_t)*src; }
// columns A[:, J[a]], a < r, densely into out (column-major, m × r) — the local share of a gather
template <class Acc>
__global__ void k_pack_cols(const Acc A, int64_t m, const int32_t* __restrict__ J, int64_t r, double* __restrict__ out) {
  for (int64_t a = blockIdx.x; a < r; a += gridDim.x) {
    const auto col = A.col(J[a]);
    for (int64_t k = threadIdx.x; k < m; k += blockDim.x) out[a * m + k] = col.ld(k);
  }
}
__global__ void k_iota(int32_t* v, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) v[i] = (int32_t)i;
}

// x[J[i]] = P[i] for i < *r_dev, and (Jx, Px, *rx_dev) ← (J, P, *r_dev): the x-update with the
// count on the device (sharded handles)
__global__ void k_scatter_dev(const int32_t* __restrict__ J, const double* __restrict__ PJ, const int64_t* r_dev,
                              double* __restrict__ x, int32_t* __restrict__ Jx, double* __restrict__ Px,
                              int64_t* rx_dev) {
  const int64_t r = *r_dev;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = tid; i < r; i += nth) {
    const int32_t j = J[i];
    const double v = PJ[i];
    x[j] = v;
    Jx[i] = j;
    Px[i] = v;
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    *rx_dev = r;
  }
}

__global__ void k_scatter(const int32_t* __restrict__ idx, const double* __restrict__ v, int64_t cnt, double* x) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < cnt) x[idx[i]] = v[i];
}

}  // namespace ssn

// ---------------------------------------------------------------------------
// Model selection along the λ path (Section 3.3)
// ---------------------------------------------------------------------------
namespace ssn {

// Appended rows for the degrees-of-freedom factorisation: rows [row0, row0+m) of M.
//   ident = 0: C = A_J (M[row0 + k, a] = A[k, J_a], a < r)        (r < m)
//   ident = 1: C = I_m (M[row0 + k, a] = δ_ka, a < m)              (r ≥ m)
template <class Acc>
__global__ void k_fill_rows(double* __restrict__ M, int64_t ld, int64_t row0, const Acc A,
                            int64_t m, const int32_t* __restrict__ J, int64_t ncol, int ident) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m * ncol) return;
  const int64_t k = e % m, a = e / m;
  M[row0 + k + a * ld] = ident ? (k == a ? 1.0 : 0.0) : A.ld(J[a], k);
}

// Deterministic Σ M[row0+i, j]² over i < nr, j < nc (single CTA, fixed per-thread order + tree).
__global__ void __launch_bounds__(1024) k_frob(const double* __restrict__ M, int64_t ld, int64_t row0, int64_t nr,
                                               int64_t nc, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t e = threadIdx.x; e < nr * nc; e += blockDim.x) {
    const double v = M[row0 + e % nr + (e / nr) * ld];
    s += v * v;
  }
  s = warp_allsum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    *out = t;
  }
}

// ν from the Frobenius sum, rss from the residual, then Eq. (21): out = [ν, rss, gcv, ebic].
//   r < m:  ν = ‖A_J L⁻ᵀ‖_F²;   r ≥ m: ν = m − λ2 ‖L⁻¹‖_F²   (push-through identity)
__global__ void k_criteria(const double* __restrict__ frob, int ident, double l2, const double* __restrict__ resid,
                           int64_t m, int64_t n, const int* ols_info, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t k = threadIdx.x; k < m; k += blockDim.x) s += resid[k] * resid[k];
  s = warp_allsum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double rss = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) rss += red[w];
    if (ols_info == nullptr || *ols_info != 0) rss = nan("");  // OLS undefined / not positive definite
    const double dm = (double)m;
    const double nu = ident ? dm - l2 * (*frob) : *frob;
    const double f = 1.0 - nu / dm;
    out[0] = nu;
    out[1] = rss;
    out[2] = (rss / dm) / (f * f);
    out[3] = log(rss / dm) + (nu / dm) * (log(dm) + log((double)n));
  }
}

}  // namespace ssn
