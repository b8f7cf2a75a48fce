// k_newton.cuh — the generalized-Hessian system V d = −∇ψ, V = I_m + κ A_J A_Jᵀ
// (Eq. (16)-(18)), with the Sherman–Morrison–Woodbury form Eq. (19)
// when r < m.  All products read the active columns A[:, J[a]] in place
// (each column is m contiguous doubles); nothing is gathered into a copy.
//
// K2  k_gather_axpy    : per-CTA partials of Σ_a coef_a A[:, J_a]          (A_J v, A_J P_J)
//     k_combine        : out = bs·base + Σ parts (fixed order), optional dot
//     k_jt_gemv        : u = A_Jᵀ g                                          (SMW rhs)
// K3  k_gram_smw       : κ⁻¹ I_r + A_JᵀA_J  (lower, r × r)                   Eq. (19)
//     k_gram_mm        : split-K partials of A_J A_Jᵀ (lower tiles, m × m)    Eq. (18)
//     k_gram_mm_reduce : I_m + κ Σ_splits
// K4  k_chol_cluster   : blocked right-looking Cholesky by one thread-block cluster,
//                        tiles in L2, cluster barriers between panel phases
//     k_chol_solve     : L Lᵀ v = rhs (single CTA), optional scale and gᵀd
#pragma once
#include <cooperative_groups.h>
#include "common.cuh"

namespace ssn {

// ---------------------------------------------------------------------------
// K2: part_vec[b][k] = Σ_{a ∈ chunk b} coef[a] * A[k, J[a]]
// ---------------------------------------------------------------------------
template <int MR>
__global__ void __launch_bounds__(256) k_gather_axpy(const double* __restrict__ A, int64_t m,
                                                     const int32_t* __restrict__ J, const double* __restrict__ coef,
                                                     int64_t r, double* __restrict__ part_vec) {
  extern __shared__ double red[];  // 8 x m
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t a_lo = (int64_t)blockIdx.x * r / gridDim.x, a_hi = (int64_t)(blockIdx.x + 1) * r / gridDim.x;
  double acc[MR];
#pragma unroll
  for (int t = 0; t < MR; ++t) acc[t] = 0.0;
  for (int64_t a = a_lo + warp; a < a_hi; a += 8) {
    const double* col = A + (int64_t)J[a] * m;
    const double c = coef[a];
#pragma unroll
    for (int t = 0; t < MR; ++t) {
      const int64_t row = lane + 32 * t;
      if (row < m) acc[t] = fma(c, __ldg(col + row), acc[t]);
    }
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

// out[k] = bs*base[k] + Σ_{b<nparts} parts[b][k] (b ascending); if dotv: *dot_out = Σ dotv·out
__global__ void __launch_bounds__(1024) k_combine(int64_t m, const double* __restrict__ base, double bs,
                                                  const double* __restrict__ parts, int nparts,
                                                  double* __restrict__ out, const double* __restrict__ dotv,
                                                  double* dot_out) {
  __shared__ double red[32];
  const int tid = threadIdx.x;
  double dot = 0.0;
  for (int64_t k = tid; k < m; k += blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nparts; ++b) s += parts[(size_t)b * m + k];
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

// u[a] = Σ_k A[k, J[a]] g[k]   (one warp per column)
__global__ void __launch_bounds__(256) k_jt_gemv(const double* __restrict__ A, int64_t m,
                                                 const int32_t* __restrict__ J, int64_t r,
                                                 const double* __restrict__ g, double* __restrict__ u) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t a = wid; a < r; a += nw) {
    const double* col = A + (int64_t)J[a] * m;
    double s = 0.0;
    for (int64_t k = lane; k < m; k += 32) s = fma(__ldg(col + k), g[k], s);
    s = warp_allsum(s);
    if (lane == 0) u[a] = s;
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

// M[a + b*r] = Σ_k A[k,J_a] A[k,J_b] (+ kinv if a == b), a ≥ b
__global__ void __launch_bounds__(256) k_gram_smw(const double* __restrict__ A, int64_t m,
                                                  const int32_t* __restrict__ J, int r, double kinv,
                                                  double* __restrict__ M) {
  __shared__ double sA[32][33], sB[32][33];
  int ti, tj;
  tri_tile(blockIdx.x, &ti, &tj);
  const int a0 = ti * 32, b0 = tj * 32;
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  double acc[4] = {0, 0, 0, 0};
  for (int64_t k0 = 0; k0 < m; k0 += 32) {
    for (int e = tid; e < 1024; e += 256) {
      const int col = e >> 5, row = e & 31;
      const int64_t k = k0 + row;
      sA[row][col] = (a0 + col < r && k < m) ? __ldg(A + (int64_t)J[a0 + col] * m + k) : 0.0;
      sB[row][col] = (b0 + col < r && k < m) ? __ldg(A + (int64_t)J[b0 + col] * m + k) : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < 32; ++kk) {
      const double bv = sB[kk][tx];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = fma(sA[kk][ty * 4 + q], bv, acc[q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int a = a0 + ty * 4 + q, b = b0 + tx;
    if (a < r && b < r && a >= b) M[(int64_t)a + (int64_t)b * r] = acc[q] + (a == b ? kinv : 0.0);
  }
}

// W[s][k + l*m] = Σ_{a in split s} A[k,J_a] A[l,J_a], k ≥ l (lower tiles)
__global__ void __launch_bounds__(256) k_gram_mm(const double* __restrict__ A, int64_t m,
                                                 const int32_t* __restrict__ J, int64_t r,
                                                 double* __restrict__ W) {
  __shared__ double sA[32][33], sB[32][33];
  int ti, tj;
  tri_tile(blockIdx.x, &ti, &tj);
  const int64_t k0 = ti * 32, l0 = tj * 32;
  const int s = blockIdx.y, ns = gridDim.y;
  const int64_t a_lo = (int64_t)s * r / ns, a_hi = (int64_t)(s + 1) * r / ns;
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  double acc[4] = {0, 0, 0, 0};
  for (int64_t a0 = a_lo; a0 < a_hi; a0 += 32) {
    for (int e = tid; e < 1024; e += 256) {
      const int ac = e >> 5, row = e & 31;  // column a0+ac, row offset
      const bool ok = a0 + ac < a_hi;
      const double* col = ok ? A + (int64_t)J[a0 + ac] * m : A;
      sA[ac][row] = (ok && k0 + row < m) ? __ldg(col + k0 + row) : 0.0;
      sB[ac][row] = (ok && l0 + row < m) ? __ldg(col + l0 + row) : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int aa = 0; aa < 32; ++aa) {
      const double bv = sB[aa][tx];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = fma(sA[aa][ty * 4 + q], bv, acc[q]);
    }
    __syncthreads();
  }
  double* Ws = W + (size_t)s * m * m;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int64_t k = k0 + ty * 4 + q, l = l0 + tx;
    if (k < m && l < m && k >= l) Ws[k + l * m] = acc[q];
  }
}

// M[k + l*m] = (k == l) + κ Σ_s W[s][k + l*m]   (k ≥ l)
__global__ void k_gram_mm_reduce(const double* __restrict__ W, int ns, int64_t m, double kappa,
                                 double* __restrict__ M) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m * m) return;
  const int64_t k = e % m, l = e / m;
  if (k < l) return;
  double s = 0.0;
  for (int q = 0; q < ns; ++q) s += W[(size_t)q * m * m + e];
  M[e] = kappa * s + (k == l ? 1.0 : 0.0);
}

// ---------------------------------------------------------------------------
// K4: Cholesky by one cluster.  M is N × N column-major (ld), lower used/overwritten.
// Right-looking, 32 × 32 tiles kept in L2 (__ldcg), per panel k:
//   B: L_ik = A_ik L_kk^{-T} for i > k           (warp per tile, all CTAs)   | cluster barrier
//   C: A_ij −= L_ik L_jkᵀ for k < j ≤ i           (warp per tile, all CTAs)   | cluster barrier
//      look-ahead: the warp that updates tile (k+1, k+1) factors it right away,
//      so panel k+1 needs no separate diagonal phase.
// ---------------------------------------------------------------------------
constexpr int CHT = 32;  // tile edge

// Factor the 32×32 tile (k0, kn) of M in registers (lane = row), write L back.
SSN_DEV void chol_diag_warp(double* M, int ld, int k0, int kn, int lane, int* info) {
  double a[CHT];
#pragma unroll
  for (int c = 0; c < CHT; ++c)
    a[c] = (lane < kn && c < kn) ? __ldcg(M + (int64_t)(k0 + lane) + (int64_t)(k0 + c) * ld)
                                 : (lane == c ? 1.0 : 0.0);
#pragma unroll
  for (int j = 0; j < CHT; ++j) {
    double ajj = __shfl_sync(0xffffffffu, a[j], j);
    if (!(ajj > 0.0)) {
      if (lane == 0) atomicExch(info, 1);
      ajj = 1.0;
    }
    const double d = sqrt(ajj);
    const double inv = 1.0 / d;
    const double lij = (lane > j) ? a[j] * inv : (lane == j ? d : 0.0);
    a[j] = lij;
#pragma unroll
    for (int c = j + 1; c < CHT; ++c) {
      const double lcj = __shfl_sync(0xffffffffu, lij, c);
      if (lane >= c) a[c] = fma(-lij, lcj, a[c]);
    }
  }
  if (lane < kn) {
#pragma unroll
    for (int c = 0; c < CHT; ++c)
      if (c <= lane && c < kn) M[(int64_t)(k0 + lane) + (int64_t)(k0 + c) * ld] = a[c];
  }
}

__global__ void __launch_bounds__(256, 1) k_chol_cluster(double* M, int N, int ld, int* info) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank(), CS = (int)cl.num_blocks();
  extern __shared__ double dsm[];
  double(*D)[33] = reinterpret_cast<double(*)[33]>(dsm);  // L_kk
  double* invd = dsm + 32 * 33;                            // 1 / L_kk[c][c]
  double* wsm = invd + 32;                                 // 8 warps x 32 x 32
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nt = (N + CHT - 1) / CHT;
  const int gw = rank + CS * warp;  // global warp id in the cluster
  const int NWg = CS * 8;

  if (gw == 0) chol_diag_warp(M, ld, 0, min(CHT, N), lane, info);
  cl.sync();
  for (int k = 0; k + 1 < nt; ++k) {
    const int k0 = k * CHT;  // kn = 32 for every panel but the last
    // ---- B: L_ik = A_ik L_kk^{-T}, i > k ----
    const int ntiles = nt - k - 1;
    if (rank < ntiles) {  // CTAs with at least one tile load L_kk
      for (int e = tid; e < CHT * CHT; e += blockDim.x) {
        const int i = e & 31, j = e >> 5;
        D[i][j] = (i >= j) ? __ldcg(M + (int64_t)(k0 + i) + (int64_t)(k0 + j) * ld) : 0.0;
      }
      __syncthreads();
      if (tid < CHT) invd[tid] = 1.0 / D[tid][tid];
      __syncthreads();
      for (int q = gw; q < ntiles; q += NWg) {
        const int row = (k + 1 + q) * CHT + lane;
        double x[CHT];
#pragma unroll
        for (int c = 0; c < CHT; ++c) x[c] = (row < N) ? __ldcg(M + (int64_t)row + (int64_t)(k0 + c) * ld) : 0.0;
#pragma unroll
        for (int c = 0; c < CHT; ++c) {
          double s0 = x[c], s1 = 0.0;
#pragma unroll
          for (int p = 0; p < c; ++p) {
            if (p & 1) s1 = fma(-x[p], D[c][p], s1);
            else s0 = fma(-x[p], D[c][p], s0);
          }
          x[c] = (s0 + s1) * invd[c];
        }
        if (row < N) {
#pragma unroll
          for (int c = 0; c < CHT; ++c) M[(int64_t)row + (int64_t)(k0 + c) * ld] = x[c];
        }
      }
    }
    cl.sync();
    // ---- C: A_ij −= L_ik L_jkᵀ, k < j ≤ i; tile (k+1,k+1) first, then factored ----
    {
      const int rem = nt - k - 1;
      const int npairs = rem * (rem + 1) / 2;
      double* S = wsm + (size_t)warp * CHT * CHT;  // S[p*32 + l] = L_jk[l][p]
      for (int q = gw; q < npairs; q += NWg) {
        int ii, jj;
        tri_tile(q, &ii, &jj);  // q = 0 → (0,0) = tile (k+1, k+1)
        const int i0 = (k + 1 + ii) * CHT, j0 = (k + 1 + jj) * CHT;
        const int row = i0 + lane;
        double a[CHT];
#pragma unroll
        for (int p = 0; p < CHT; ++p) {
          a[p] = (row < N) ? __ldcg(M + (int64_t)row + (int64_t)(k0 + p) * ld) : 0.0;
          S[p * CHT + lane] = (j0 + lane < N) ? __ldcg(M + (int64_t)(j0 + lane) + (int64_t)(k0 + p) * ld) : 0.0;
        }
        __syncwarp();
        double c[CHT];
#pragma unroll
        for (int l = 0; l < CHT; ++l)
          c[l] = (row < N && j0 + l < N) ? __ldcg(M + (int64_t)row + (int64_t)(j0 + l) * ld) : 0.0;
#pragma unroll
        for (int p = 0; p < CHT; ++p) {
          const double ap = a[p];
          const double2* Sp = reinterpret_cast<const double2*>(S + p * CHT);
#pragma unroll
          for (int l2 = 0; l2 < CHT / 2; ++l2) {
            const double2 sv = Sp[l2];
            c[2 * l2] = fma(-ap, sv.x, c[2 * l2]);
            c[2 * l2 + 1] = fma(-ap, sv.y, c[2 * l2 + 1]);
          }
        }
        if (row < N) {
#pragma unroll
          for (int l = 0; l < CHT; ++l)
            if (j0 + l < N && (i0 != j0 || l <= lane)) M[(int64_t)row + (int64_t)(j0 + l) * ld] = c[l];
        }
        __syncwarp();
        if (q == 0) {  // look-ahead: factor the next diagonal tile now
          __threadfence_block();
          chol_diag_warp(M, ld, (k + 1) * CHT, min(CHT, N - (k + 1) * CHT), lane, info);
        }
      }
    }
    cl.sync();
  }
}

// Solve (L Lᵀ) v = rhs; out = scale * v; if dotv: *dot_out = Σ dotv · out.  Single CTA, N ≤ 4096.
__global__ void __launch_bounds__(1024) k_chol_solve(const double* __restrict__ L, int N, int ld,
                                                     const double* __restrict__ rhs, double scale,
                                                     double* __restrict__ out, const double* __restrict__ dotv,
                                                     double* dot_out) {
  extern __shared__ double z[];
  __shared__ double red[32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < N; i += blockDim.x) z[i] = rhs[i];
  __syncthreads();
  // forward: L y = z
  for (int k0 = 0; k0 < N; k0 += 32) {
    const int kn = min(32, N - k0);
    if (warp == 0) {
      const int c = lane;
      double Lr[32];
#pragma unroll
      for (int p = 0; p < 32; ++p) Lr[p] = (c < kn && p < c) ? L[(int64_t)(k0 + c) + (int64_t)(k0 + p) * ld] : 0.0;
      const double dinv = (c < kn) ? 1.0 / L[(int64_t)(k0 + c) * (ld + 1)] : 1.0;
      double zc = (c < kn) ? z[k0 + c] : 0.0;
#pragma unroll
      for (int p = 0; p < 32; ++p) {
        if (lane == p) zc *= dinv;
        const double zp = __shfl_sync(0xffffffffu, zc, p);
        if (lane > p) zc = fma(-Lr[p], zp, zc);
      }
      if (c < kn) z[k0 + c] = zc;
    }
    __syncthreads();
    for (int i = k0 + kn + tid; i < N; i += blockDim.x) {
      double s = 0.0;
      for (int p = 0; p < kn; ++p) s = fma(L[(int64_t)i + (int64_t)(k0 + p) * ld], z[k0 + p], s);
      z[i] -= s;
    }
    __syncthreads();
  }
  // backward: Lᵀ v = y
  const int nb = (N + 31) / 32;
  for (int kb = nb - 1; kb >= 0; --kb) {
    const int k0 = kb * 32, kn = min(32, N - k0);
    if (warp == 0) {
      const int c = lane;
      double Lc[32];  // Lc[p] = L[k0+p][k0+c] for p > c
#pragma unroll
      for (int p = 0; p < 32; ++p)
        Lc[p] = (c < kn && p < kn && p > c) ? L[(int64_t)(k0 + p) + (int64_t)(k0 + c) * ld] : 0.0;
      const double dinv = (c < kn) ? 1.0 / L[(int64_t)(k0 + c) * (ld + 1)] : 1.0;
      double zc = (c < kn) ? z[k0 + c] : 0.0;
#pragma unroll
      for (int p = 31; p >= 0; --p) {
        if (lane == p) zc *= dinv;
        const double zp = __shfl_sync(0xffffffffu, zc, p);
        if (lane < p) zc = fma(-Lc[p], zp, zc);
      }
      if (c < kn) z[k0 + c] = zc;
    }
    __syncthreads();
    for (int i = tid; i < k0; i += blockDim.x) {
      double s = 0.0;
      const double* Lcol = L + (int64_t)i * ld + k0;  // L[k0+p][i]
      for (int p = 0; p < kn; ++p) s = fma(Lcol[p], z[k0 + p], s);
      z[i] -= s;
    }
    __syncthreads();
  }
  double dot = 0.0;
  for (int i = tid; i < N; i += blockDim.x) {
    const double v = scale * z[i];
    out[i] = v;
    if (dotv) dot += dotv[i] * v;
  }
  if (dotv) {
    dot = warp_allsum(dot);
    if (lane == 0) red[warp] = dot;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int wi = 0; wi < (int)(blockDim.x >> 5); ++wi) s += red[wi];
      *dot_out = s;
    }
  }
}

// y ← y + s·d  (m-vector) and small helpers
__global__ void k_axpy_m(int64_t m, const double* y, double s, const double* d, double* out) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < m) out[k] = __dadd_rn(y[k], __dmul_rn(s, d[k]));
}
__global__ void k_neg_copy(int64_t m, const double* g, double* d, const double* dotv, double* dot_out) {
  __shared__ double red[32];
  double dot = 0.0;
  for (int64_t k = threadIdx.x; k < m; k += blockDim.x) {
    d[k] = -g[k];
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
__global__ void k_zero_at(const int32_t* __restrict__ idx, int64_t cnt, double* x) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < cnt) x[idx[i]] = 0.0;
}
__global__ void k_scatter(const int32_t* __restrict__ idx, const double* __restrict__ v, int64_t cnt, double* x) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < cnt) x[idx[i]] = v[i];
}

}  // namespace ssn
