// Probe: per-pivot cost of the 4-warp diagonal factor (diag_factor4) and variants with parts
// removed (timing only; the variants are not correct factorisations).
#include <cstdio>
#define SSN_DEV __device__ __forceinline__
constexpr int CHT = 32, TLD = 33;
SSN_DEV double sel8(const double (&v)[8], int i) {
  double r = v[0];
#pragma unroll
  for (int q = 1; q < 8; ++q) r = (i == q) ? v[q] : r;
  return r;
}
template <int V>
__global__ void k_diag(const double* Sg, double* out, unsigned long long* cyc) {
  __shared__ double S[CHT * TLD + 80];
  const int t128 = threadIdx.x, w = t128 >> 5, lane = t128 & 31;
  for (int e = t128; e < CHT * TLD; e += 128) S[e] = Sg[e];
  __syncthreads();
  double* cb = S + CHT * TLD;
  const int kn = 32, nrow = 32;
  long long c0 = clock64();
  double a[8], dgw[8], wv[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int c = 8 * w + q;
    a[q] = (lane < nrow && c < kn) ? S[lane * TLD + c] : (lane == c ? 1.0 : 0.0);
    dgw[q] = (c < kn) ? S[c * TLD + c] : 1.0;
    wv[q] = (lane == c) ? 1.0 : 0.0;
  }
  bool bad = false;
#pragma unroll 1
  for (int j = 0; j < CHT; ++j) {
    double* cbj = cb + (j & 1) * 33;
    const int jl = j & 7;
    if (w == (j >> 3)) {
      double d = sel8(dgw, jl);
      bad |= (j < kn) && !(d > 0.0);
      d = (j < kn && d > 0.0) ? d : 1.0;
      const double inv = (V == 1) ? d : rsqrt(d);
      const double aj = sel8(a, jl);
      const double lij = (lane > j) ? aj * inv : (lane == j ? d * inv : 0.0);
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] = (q == jl) ? lij : a[q];
      cbj[lane] = lij;
      if (lane == 0) cbj[32] = inv;
    }
    if (V != 3) asm volatile("bar.sync 2, 128;" ::: "memory");
    const double li = cbj[lane], inv = cbj[32];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int c = 8 * w + q;
      const double lc = (c > j) ? cbj[c] : 0.0;
      a[q] = fma(-li, lc, a[q]);
      dgw[q] = fma(-lc, lc, dgw[q]);
      if (V != 2) {
        const double wj = __shfl_sync(0xffffffffu, wv[q], j) * inv;
        wv[q] = (lane == j) ? wj : ((lane > j) ? fma(-li, wj, wv[q]) : wv[q]);
      }
    }
  }
  long long c1 = clock64();
  double s = bad ? 1.0 : 0.0;
  for (int q = 0; q < 8; ++q) s += a[q] + dgw[q] + wv[q];
  out[t128] = s;
  if (t128 == 0) cyc[V] = c1 - c0;
}
__global__ void k_rsqrt_chain(double* out, unsigned long long* cyc) {
  double x = 2.0 + threadIdx.x;
  long long c0 = clock64();
  for (int i = 0; i < 1000; ++i) x = rsqrt(x) + 1.5;
  long long c1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[8] = c1 - c0;
}
__global__ void k_bar_pingpong(double* out, unsigned long long* cyc) {  // owner writes, bar, all read
  __shared__ double cb[66];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double v = lane;
  long long c0 = clock64();
#pragma unroll 1
  for (int j = 0; j < 1000; ++j) {
    double* c = cb + (j & 1) * 33;
    if (w == ((j >> 3) & 3)) c[lane] = v * 1.0000001;
    asm volatile("bar.sync 2, 128;" ::: "memory");
    v = c[lane] + c[(lane + 1) & 31];
  }
  long long c1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) cyc[9] = c1 - c0;
}
int main() {
  double h[CHT * TLD];
  for (int r = 0; r < CHT; ++r)
    for (int c = 0; c < TLD; ++c) h[r * TLD + c] = (r == c) ? 40.0 : ((c < CHT) ? 0.01 * ((r * 7 + c * 13) % 11) : 0.0);
  for (int r = 0; r < CHT; ++r) for (int c = 0; c < r; ++c) h[c * TLD + r] = h[r * TLD + c];
  double *dS, *o; unsigned long long* cyc;
  cudaMalloc(&dS, sizeof(h)); cudaMalloc(&o, 4096); cudaMalloc(&cyc, 128);
  cudaMemcpy(dS, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 2; ++rep) {
    k_diag<0><<<1, 128>>>(dS, o, cyc);
    k_diag<1><<<1, 128>>>(dS, o, cyc);
    k_diag<2><<<1, 128>>>(dS, o, cyc);
    k_diag<3><<<1, 128>>>(dS, o, cyc);
    k_rsqrt_chain<<<1, 32>>>(o, cyc);
    k_bar_pingpong<<<1, 128>>>(o, cyc);
    cudaDeviceSynchronize();
  }
  unsigned long long c[10];
  cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  printf("full %llu cyc (%.0f/pivot); no-rsqrt %llu; no-W %llu; no-bar %llu\n", c[0], c[0] / 32.0, c[1], c[2], c[3]);
  printf("rsqrt chain %.1f cyc/iter; owner-write+bar(128)+read ping-pong %.1f cyc/iter\n", c[8] / 1000.0, c[9] / 1000.0);
  return 0;
}
