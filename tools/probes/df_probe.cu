// Probe: variants of the 32 x 32 diagonal factor (W on/off, Newton steps of the reciprocal sqrt).
#include <cstdio>
#include <cmath>
#include "../../paper_2006_03970_b200/csrc/k_newton.cuh"
using namespace ssn;
template <int NEWTON> __device__ __forceinline__ double rsq_n(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
#pragma unroll
  for (int it = 0; it < NEWTON; ++it) { const double r = fma(-d * y, y, 1.0); y = fma(0.5 * y, r, y); }
  return y;
}
template <bool WANTW, int NEWTON>
__device__ __forceinline__ void df_var(const double* S, double* M, int ld, int n0, int kn, int nrow, double* Wout, double* Wsm,
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
            if (WANTW) wr[p] = fma(-l, wbp[pp], wr[p]);
          }
      }
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int j = 8 * blk + p;
        double d = dgw[p];
        bad |= (j < kn) && !(d > 0.0);
        d = (j < kn && d > 0.0) ? d : 1.0;
        const double inv = rsq_n<NEWTON>(d);
        const double lij = (lane > j) ? a[p] * inv : (lane == j ? d * inv : 0.0);
        const double wj = wr[p] * inv;  // W row j scaled (final)
#pragma unroll
        for (int q = p + 1; q < 8; ++q) {
          const double lq = __shfl_sync(0xffffffffu, lij, 8 * blk + q);  // L[8blk+q][j]
          dgw[q] = fma(-lq, lq, dgw[q]);
          a[q] = fma(-lij, lq, a[q]);
          if (WANTW) wr[q] = fma(-lq, wj, wr[q]);
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
          if (WANTW) wr[q] = fma(-l, wb[p], wr[q]);
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


// one warp, lane = row, the row in registers, fully unrolled (L only)
template <int NEWTON>
__device__ __forceinline__ void df_warp(double* S, int lane) {
  double a0[CHT];
#pragma unroll
  for (int c = 0; c < CHT; ++c) a0[c] = S[lane * TLD + c];
  double d = __shfl_sync(0xffffffffu, a0[0], 0);
#pragma unroll
  for (int j = 0; j < CHT; ++j) {
    const double dd = d > 0.0 ? d : 1.0;
    const double inv = rsq_n<NEWTON>(dd);
    const double l0 = lane > j ? a0[j] * inv : (lane == j ? dd * inv : 0.0);
    a0[j] = l0;
    if (j + 1 < CHT) {
      const double lq = __shfl_sync(0xffffffffu, l0, j + 1);
      a0[j + 1] = fma(-l0, lq, a0[j + 1]);
      d = __shfl_sync(0xffffffffu, a0[j + 1], j + 1);
    }
#pragma unroll
    for (int q = j + 2; q < CHT; ++q) {
      const double lq = __shfl_sync(0xffffffffu, l0, q);
      a0[q] = fma(-l0, lq, a0[q]);
    }
  }
#pragma unroll
  for (int c = 0; c < CHT; ++c) S[lane * TLD + c] = c <= lane ? a0[c] : 0.0;
}
template <int NEWTON>
__global__ void k_warp(const double* Sg, double* M, unsigned long long* cyc) {
  __shared__ double S[CHT * TLD];
  for (int e = threadIdx.x; e < CHT * TLD; e += 32) S[e] = Sg[e];
  __syncwarp();
  long long c0 = clock64();
  df_warp<NEWTON>(S, threadIdx.x);
  long long c1 = clock64();
  if (threadIdx.x == 0) cyc[0] = c1 - c0;
  for (int e = threadIdx.x; e < CHT * CHT; e += 32) M[e] = S[(e % 32) * TLD + e / 32];
}

// L-only variant: the next owner applies the previous block's rank-8 update lazily, column by
// column right before each pivot, with two partial sums (shorter chains); no W.
template <int NEWTON>
__device__ __forceinline__ void df_lazy(double* S, double* cb, int t128) {
  const int w = t128 >> 5, lane = t128 & 31;
  constexpr int BS = CHT * 9;
  double a[8], dgw[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int c = 8 * w + q;
    a[q] = S[lane * TLD + c];
    dgw[q] = S[c * TLD + c];
  }
#pragma unroll 1
  for (int blk = 0; blk < 4; ++blk) {
    double* Lb = cb + (blk & 1) * BS;
    if (w == blk) {
      const double* Lp = cb + ((blk + 1) & 1) * BS;
      double lrp[8];
      if (blk > 0)
#pragma unroll
        for (int pp = 0; pp < 8; ++pp) lrp[pp] = Lp[lane * 9 + pp];
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        if (blk > 0) {
          double d0 = 0, d1 = 0, a0 = 0, a1 = 0;
#pragma unroll
          for (int pp = 0; pp < 8; pp += 2) {
            const double l0 = Lp[(8 * w + p) * 9 + pp], l1 = Lp[(8 * w + p) * 9 + pp + 1];
            d0 = fma(l0, l0, d0); d1 = fma(l1, l1, d1);
            a0 = fma(lrp[pp], l0, a0); a1 = fma(lrp[pp + 1], l1, a1);
          }
          dgw[p] -= d0 + d1;
          a[p] -= a0 + a1;
        }
        const int j = 8 * blk + p;
        double d = dgw[p];
        d = d > 0.0 ? d : 1.0;
        const double inv = rsq_n<NEWTON>(d);
        const double lij = (lane > j) ? a[p] * inv : (lane == j ? d * inv : 0.0);
#pragma unroll
        for (int q = p + 1; q < 8; ++q) {
          const double lq = __shfl_sync(0xffffffffu, lij, 8 * blk + q);
          dgw[q] = fma(-lq, lq, dgw[q]);
          a[q] = fma(-lij, lq, a[q]);
        }
        a[p] = lij;
      }
#pragma unroll
      for (int p = 0; p < 8; ++p) Lb[lane * 9 + p] = a[p];
    }
    asm volatile("bar.sync 2, 128;" ::: "memory");
    if (w > blk + 1) {
      double lr[8];
#pragma unroll
      for (int p = 0; p < 8; ++p) lr[p] = Lb[lane * 9 + p];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const double* lc = Lb + (8 * w + q) * 9;
#pragma unroll
        for (int p = 0; p < 8; ++p) {
          const double l = lc[p];
          dgw[q] = fma(-l, l, dgw[q]);
          a[q] = fma(-lr[p], l, a[q]);
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int c = 8 * w + q;
    S[lane * TLD + c] = c <= lane ? a[q] : 0.0;
  }
}
template <int NEWTON>
__global__ void k_lazy(const double* Sg, double* M, unsigned long long* cyc) {
  __shared__ double S[CHT * TLD + kDiagScratch];
  for (int e = threadIdx.x; e < CHT * TLD; e += 128) S[e] = Sg[e];
  __syncthreads();
  long long c0 = clock64();
  df_lazy<NEWTON>(S, S + CHT * TLD, threadIdx.x);
  long long c1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[0] = c1 - c0;
  for (int e = threadIdx.x; e < CHT * CHT; e += 128) M[e] = S[(e % 32) * TLD + e / 32];
}

// chain probe: one warp does 32 pivots as 4 blocks of 8 (no rank-8 updates, no barriers, no W)
template <int MODE>
__global__ void k_chain(const double* Sg, double* M, unsigned long long* cyc) {
  const int lane = threadIdx.x;
  double a[8], dgw[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) { a[q] = Sg[lane * TLD + q]; dgw[q] = Sg[q * TLD + q]; }
  long long c0 = clock64();
#pragma unroll 1
  for (int blk = 0; blk < 4; ++blk) {
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      const int j = 8 * blk + p;
      double d = dgw[p];
      d = d > 0.0 ? d : 1.0;
      double inv;
      if (MODE == 0) inv = rsq_n<2>(d);
      else if (MODE == 1) inv = rsq_n<0>(d);
      else inv = 1.0 / sqrt(d);
      const double lij = (lane > j) ? a[p] * inv : (lane == j ? d * inv : 0.0);
#pragma unroll
      for (int q = p + 1; q < 8; ++q) {
        const double lq = __shfl_sync(0xffffffffu, lij, 8 * blk + q);
        dgw[q] = fma(-lq, lq, dgw[q]);
        a[q] = fma(-lij, lq, a[q]);
      }
      a[p] = lij;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) { dgw[q] = dgw[q] * 0.5 + 4.0; }
  }
  long long c1 = clock64();
  if (lane == 0) cyc[0] = c1 - c0;
  for (int q = 0; q < 8; ++q) M[lane * 8 + q] = a[q];
}
template <int NW>
__device__ __forceinline__ void df_nw(const double* S, double* M, int ld, int n0, int kn, int nrow, double* Wout, double* Wsm,
                          int* info, double* cb, int t128) {
  constexpr int BC = 32 / NW;
  const int w = t128 >> 5, lane = t128 & 31;
  double a[BC], dgw[BC], wr[BC];
#pragma unroll
  for (int q = 0; q < BC; ++q) {
    const int c = BC * w + q;
    a[q] = (lane < nrow && c < kn) ? S[lane * TLD + c] : (lane == c ? 1.0 : 0.0);
    dgw[q] = (c < kn) ? S[c * TLD + c] : 1.0;
    wr[q] = (lane == c) ? 1.0 : 0.0;
  }
  bool bad = false;
#pragma unroll 1
  for (int blk = 0; blk < NW; ++blk) {
    double* Lb = cb + (blk & 1) * (CHT * 9 + 8 * 33);  // Lb[r * 9 + p] = L[r][BC blk + p]
    double* Wb = Lb + CHT * 9;                          // Wb[p * 33 + c] = W[8blk + p][c]
    if (w == blk) {
      const double* Lp = cb + ((blk + 1) & 1) * (CHT * 9 + 8 * 33);  // block blk − 1
      const double* Wp = Lp + CHT * 9;
      double lrp[BC], wbp[BC];
      if (blk > 0) {
#pragma unroll
        for (int pp = 0; pp < BC; ++pp) {
          lrp[pp] = Lp[lane * 9 + pp];
          wbp[pp] = Wp[pp * 33 + lane];
        }
      }
      if (blk > 0) {  // rank-8 update of this block's columns from block blk − 1, before any pivot:
                      // eight independent chains, so only pivot 0 waits for one of them
#pragma unroll
        for (int p = 0; p < BC; ++p)
#pragma unroll
          for (int pp = 0; pp < BC; ++pp) {
            const double l = Lp[(BC * w + p) * 9 + pp];
            dgw[p] = fma(-l, l, dgw[p]);
            a[p] = fma(-lrp[pp], l, a[p]);
            wr[p] = fma(-l, wbp[pp], wr[p]);
          }
      }
#pragma unroll
      for (int p = 0; p < BC; ++p) {
        const int j = BC * blk + p;
        double d = dgw[p];
        bad |= (j < kn) && !(d > 0.0);
        d = (j < kn && d > 0.0) ? d : 1.0;
        const double inv = rsq_n<2>(d);
        const double lij = (lane > j) ? a[p] * inv : (lane == j ? d * inv : 0.0);
        const double wj = wr[p] * inv;  // W row j scaled (final)
#pragma unroll
        for (int q = p + 1; q < BC; ++q) {
          const double lq = __shfl_sync(0xffffffffu, lij, BC * blk + q);  // L[8blk+q][j]
          dgw[q] = fma(-lq, lq, dgw[q]);
          a[q] = fma(-lij, lq, a[q]);
          wr[q] = fma(-lq, wj, wr[q]);
        }
        a[p] = lij;
        wr[p] = wj;
      }
#pragma unroll
      for (int p = 0; p < BC; ++p) {
        Lb[lane * 9 + p] = a[p];
        Wb[p * 33 + lane] = wr[p];
      }
    }
    asm volatile("bar.sync 2, %0;" :: "r"(NW * 32) : "memory");
    if (w > blk + 1) {  // eager rank-8 update from block blk
      double lr[BC], wb[BC];
#pragma unroll
      for (int p = 0; p < BC; ++p) {
        lr[p] = Lb[lane * 9 + p];
        wb[p] = Wb[p * 33 + lane];
      }
#pragma unroll
      for (int q = 0; q < BC; ++q) {
        const double* lc = Lb + (BC * w + q) * 9;
#pragma unroll
        for (int p = 0; p < BC; ++p) {
          const double l = lc[p];  // L[8w+q][8blk+p]
          dgw[q] = fma(-l, l, dgw[q]);
          a[q] = fma(-lr[p], l, a[q]);
          wr[q] = fma(-l, wb[p], wr[q]);
        }
      }
    }
  }
  if (bad && lane == 0) atomicExch(info, 1);
  if (!M) asm volatile("bar.sync 2, %0;" :: "r"(NW * 32) : "memory");  // every warp has read S before L overwrites it
#pragma unroll
  for (int q = 0; q < BC; ++q) {
    const int c = BC * w + q;
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


template <int NW>
__global__ void k_nw(const double* Sg, double* M, double* W, int* info, unsigned long long* cyc) {
  __shared__ double S[CHT * TLD + kDiagScratch];
  for (int e = threadIdx.x; e < CHT * TLD; e += NW * 32) S[e] = Sg[e];
  __syncthreads();
  long long c0 = clock64();
  df_nw<NW>(S, M, 32, 0, 32, 32, W, nullptr, info, S + CHT * TLD, threadIdx.x);
  long long c1 = clock64();
  if (threadIdx.x == 0) cyc[0] = c1 - c0;
}
template <bool WANTW, int NEWTON>
__global__ void k_var(const double* Sg, double* M, double* W, int* info, unsigned long long* cyc) {
  __shared__ double S[CHT * TLD + kDiagScratch];
  for (int e = threadIdx.x; e < CHT * TLD; e += 128) S[e] = Sg[e];
  __syncthreads();
  long long c0 = clock64();
  df_var<WANTW, NEWTON>(S, M, 32, 0, 32, 32, W, nullptr, info, S + CHT * TLD, threadIdx.x);
  long long c1 = clock64();
  if (threadIdx.x == 0) cyc[0] = c1 - c0;
}
// Reciprocal-pivot chain (LDL^T-style): the Schur complement is kept UNNORMALISED inside a block, so
// the dependent chain per pivot is rcp(d) -> c*inv -> fma into the next diagonal replica (the column
// values c are shuffled before inv is known); L = a * rsqrt(d) and W = D^-1/2 U^-1 off the chain.
__device__ __forceinline__ double rcp_pos(double d) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
#pragma unroll
  for (int it = 0; it < 2; ++it) { const double e = fma(-d, y, 1.0); y = fma(y, e, y); }
  return y;
}
__device__ __forceinline__ void df_rcp(const double* S, double* M, int ld, int n0, int kn, int nrow, double* Wout,
                                       double* Wsm, int* info, double* cb, int t128) {
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
    double* Lb = cb + (blk & 1) * (CHT * 9 + 8 * 33);
    double* Wb = Lb + CHT * 9;
    if (w == blk) {
      const double* Lp = cb + ((blk + 1) & 1) * (CHT * 9 + 8 * 33);
      const double* Wp = Lp + CHT * 9;
      double lrp[8], wbp[8];
      if (blk > 0) {
#pragma unroll
        for (int pp = 0; pp < 8; ++pp) {
          lrp[pp] = Lp[lane * 9 + pp];
          wbp[pp] = Wp[pp * 33 + lane];
        }
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
        double cq[8];  // unnormalised column j at rows 8blk+q (final after pivot j-1): off the chain
#pragma unroll
        for (int q = p + 1; q < 8; ++q) cq[q] = __shfl_sync(0xffffffffu, a[p], 8 * blk + q);
        double d = dgw[p];
        bad |= (j < kn) && !(d > 0.0);
        d = (j < kn && d > 0.0) ? d : 1.0;
        const double inv = rcp_pos(d);   // the chain
        const double rs = rsqrt_pos(d);  // off the chain (L and W scaling)
        const double t = a[p] * inv;     // a_ij / d_j
#pragma unroll
        for (int q = p + 1; q < 8; ++q) {
          const double u = cq[q] * inv;  // u_qj = a_qj / d_j
          dgw[q] = fma(-cq[q], u, dgw[q]);
          a[q] = fma(-t, cq[q], a[q]);
          wr[q] = fma(-u, wr[p], wr[q]);  // rows of U^-1
        }
        a[p] = (lane > j) ? a[p] * rs : (lane == j ? d * rs : 0.0);
        wr[p] = wr[p] * rs;  // W row j = rsqrt(d_j) * (U^-1 row j)
      }
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        Lb[lane * 9 + p] = a[p];
        Wb[p * 33 + lane] = wr[p];
      }
    }
    asm volatile("bar.sync 2, 128;" ::: "memory");
    if (w > blk + 1) {
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
          const double l = lc[p];
          dgw[q] = fma(-l, l, dgw[q]);
          a[q] = fma(-lr[p], l, a[q]);
          wr[q] = fma(-l, wb[p], wr[q]);
        }
      }
    }
  }
  if (bad && lane == 0) atomicExch(info, 1);
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int c = 8 * w + q;
    if (lane < nrow && c < kn && c <= lane) M[(int64_t)(n0 + lane) + (int64_t)(n0 + c) * ld] = a[q];
    const double wv = (c < kn && lane < kn) ? wr[q] : (lane == c ? 1.0 : 0.0);
    if (Wout) Wout[c * CHT + lane] = wv;
  }
}
__global__ void k_rcp(const double* Sg, double* M, double* W, int* info, unsigned long long* cyc) {
  __shared__ double S[CHT * TLD + kDiagScratch];
  for (int e = threadIdx.x; e < CHT * TLD; e += 128) S[e] = Sg[e];
  __syncthreads();
  long long c0 = clock64();
  df_rcp(S, M, 32, 0, 32, 32, W, nullptr, info, S + CHT * TLD, threadIdx.x);
  long long c1 = clock64();
  if (threadIdx.x == 0) cyc[0] = c1 - c0;
}
__global__ void k_cur(const double* Sg, double* M, double* W, int* info, unsigned long long* cyc) {
  __shared__ double S[CHT * TLD + kDiagScratch];
  for (int e = threadIdx.x; e < CHT * TLD; e += 128) S[e] = Sg[e];
  __syncthreads();
  long long c0 = clock64();
  diag_factor4(S, M, 32, 0, 32, 32, W, nullptr, info, S + CHT * TLD, threadIdx.x);
  long long c1 = clock64();
  if (threadIdx.x == 0) cyc[0] = c1 - c0;
}
template <class K> void run_lw(const char* name, K kern, const double* h, double* dS, double* dM, double* dW, int* info,
                               unsigned long long* cyc) {
  for (int rep = 0; rep < 5; ++rep) kern<<<1, 128>>>(dS, dM, dW, info, cyc);
  cudaDeviceSynchronize();
  unsigned long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  double L[32 * 32], W[32 * 32];
  cudaMemcpy(L, dM, sizeof(L), cudaMemcpyDeviceToHost); cudaMemcpy(W, dW, sizeof(W), cudaMemcpyDeviceToHost);
  double e1 = 0, e2 = 0;
  for (int i = 0; i < 32; ++i) for (int j = 0; j <= i; ++j) {
    double s2 = 0; for (int p = 0; p <= j; ++p) s2 += L[i + p * 32] * L[j + p * 32];
    e1 = fmax(e1, fabs(s2 - h[i * TLD + j]));
    double t = 0; for (int p = j; p <= i; ++p) t += W[i * 32 + p] * L[p + j * 32];
    e2 = fmax(e2, fabs(t - (i == j)));
  }
  printf("%-24s %6llu cycles (%.0f per pivot) |LL'-A| %.2e |WL-I| %.2e %s\n", name, c, c / 32.0, e1, e2,
         cudaGetErrorString(cudaGetLastError()));
}
template <bool WANTW, int NEWTON> void run(const char* name, double* dS, double* dM, double* dW, int* info, unsigned long long* cyc) {
  for (int rep = 0; rep < 5; ++rep) k_var<WANTW, NEWTON><<<1, 128>>>(dS, dM, dW, info, cyc);
  cudaDeviceSynchronize();
  unsigned long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%-24s %6llu cycles (%.0f per pivot) %s\n", name, c, c / 32.0, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  double h[CHT * TLD];
  for (int r = 0; r < CHT; ++r)
    for (int c = 0; c < TLD; ++c) h[r * TLD + c] = (r == c) ? 4.0 + r : ((c < CHT) ? 0.3 * sin(r * 7.0 + c * 13.0 + (r > c ? r * c : c * r)) : 0.0);
  for (int r = 0; r < CHT; ++r) for (int c = 0; c < r; ++c) h[c * TLD + r] = h[r * TLD + c];
  double *dS, *dM, *dW; int* info; unsigned long long* cyc;
  cudaMalloc(&dS, sizeof(h)); cudaMalloc(&dM, 32 * 32 * 8); cudaMalloc(&dW, 32 * 32 * 8); cudaMalloc(&info, 4); cudaMalloc(&cyc, 64);
  cudaMemcpy(dS, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaMemset(dM, 0, 32 * 32 * 8);
  for (int k = 0; k < 3; ++k) {
    run_lw("diag_factor4 (current)", k_cur, h, dS, dM, dW, info, cyc);
    run_lw("reciprocal chain", k_rcp, h, dS, dM, dW, info, cyc);
  }
  run<true, 2>("W, 2 Newton", dS, dM, dW, info, cyc);
  run<false, 2>("no W, 2 Newton", dS, dM, dW, info, cyc);
  run<true, 1>("W, 1 Newton", dS, dM, dW, info, cyc);
  run<false, 1>("no W, 1 Newton", dS, dM, dW, info, cyc);
  for (int v = 0; v < 2; ++v) {
    for (int rep = 0; rep < 5; ++rep) { if (v == 0) k_lazy<2><<<1, 128>>>(dS, dM, cyc); else k_lazy<1><<<1, 128>>>(dS, dM, cyc); }
    cudaDeviceSynchronize();
    unsigned long long c2; cudaMemcpy(&c2, cyc, 8, cudaMemcpyDeviceToHost);
    double L2[32 * 32]; cudaMemcpy(L2, dM, sizeof(L2), cudaMemcpyDeviceToHost);
    double e2 = 0;
    for (int i = 0; i < 32; ++i) for (int j = 0; j <= i; ++j) {
      double s2 = 0; for (int p = 0; p <= j; ++p) s2 += L2[i + p * 32] * L2[j + p * 32];
      e2 = fmax(e2, fabs(s2 - h[i * TLD + j]));
    }
    printf("%-24s %6llu cycles (%.0f per pivot) err %.2e %s\n", v == 0 ? "lazy split, no W, 2N" : "lazy split, no W, 1N", c2, c2 / 32.0, e2, cudaGetErrorString(cudaGetLastError()));
  }
  for (int md = 0; md < 3; ++md) {
    for (int rep = 0; rep < 5; ++rep) { if (md == 0) k_chain<0><<<1, 32>>>(dS, dM, cyc); else if (md == 1) k_chain<1><<<1, 32>>>(dS, dM, cyc); else k_chain<2><<<1, 32>>>(dS, dM, cyc); }
    cudaDeviceSynchronize();
    unsigned long long c3; cudaMemcpy(&c3, cyc, 8, cudaMemcpyDeviceToHost);
    printf("chain only (%s): %llu cycles (%.0f per pivot)\n", md == 0 ? "rsqrt+2N" : (md == 1 ? "MUFU only" : "1/sqrt"), c3, c3 / 32.0);
  }
  for (int rep = 0; rep < 5; ++rep) k_nw<8><<<1, 256>>>(dS, dM, dW, info, cyc);
  { cudaDeviceSynchronize(); unsigned long long c8; cudaMemcpy(&c8, cyc, 8, cudaMemcpyDeviceToHost);
    double L[32 * 32], W[32 * 32];
    cudaMemcpy(L, dM, sizeof(L), cudaMemcpyDeviceToHost); cudaMemcpy(W, dW, sizeof(W), cudaMemcpyDeviceToHost);
    double e1 = 0, e2 = 0;
    for (int i = 0; i < 32; ++i) for (int j = 0; j <= i; ++j) {
      double s2 = 0; for (int p = 0; p <= j; ++p) s2 += L[i + p * 32] * L[j + p * 32];
      e1 = fmax(e1, fabs(s2 - h[i * TLD + j]));
      double t = 0; for (int p = j; p <= i; ++p) t += W[i * 32 + p] * L[p + j * 32];
      e2 = fmax(e2, fabs(t - (i == j)));
    }
    printf("%-24s %6llu cycles (%.0f per pivot) |LL'-A| %.2e |WL-I| %.2e %s\n", "8 warps x 4 columns", c8, c8 / 32.0, e1, e2, cudaGetErrorString(cudaGetLastError())); }
  for (int rep = 0; rep < 5; ++rep) k_nw<4><<<1, 128>>>(dS, dM, dW, info, cyc);
  { cudaDeviceSynchronize(); unsigned long long c4; cudaMemcpy(&c4, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-24s %6llu cycles (%.0f per pivot)\n", "4 warps x 8 (generic)", c4, c4 / 32.0); }
  for (int rep = 0; rep < 5; ++rep) k_warp<2><<<1, 32>>>(dS, dM, cyc);
  cudaDeviceSynchronize();
  unsigned long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  double L[32 * 32]; cudaMemcpy(L, dM, sizeof(L), cudaMemcpyDeviceToHost);
  double e1 = 0;
  for (int i = 0; i < 32; ++i) for (int j = 0; j <= i; ++j) {
    double s2 = 0; for (int p = 0; p <= j; ++p) s2 += L[i + p * 32] * L[j + p * 32];
    e1 = fmax(e1, fabs(s2 - h[i * TLD + j]));
  }
  printf("%-24s %6llu cycles (%.0f per pivot) err %.2e %s\n", "1 warp unrolled, L only", c, c / 32.0, e1, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
