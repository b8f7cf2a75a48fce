// Probe: cost of a dependent smem-update + __syncthreads step for 128 / 256 / 512 / 1024-thread CTAs.
#include <cstdio>
template <int T>
__global__ void k_bar(double* out, unsigned long long* cyc, int iters) {
  __shared__ double s[1024];
  s[threadIdx.x] = threadIdx.x;
  __syncthreads();
  long long c0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const double v = s[(threadIdx.x + it) & (T - 1)];
    __syncthreads();
    s[threadIdx.x] = fma(v, 1.0000001, 0.5);
    __syncthreads();
  }
  long long c1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = c1 - c0; out[0] = s[5]; }
}
int main() {
  double* o; unsigned long long* c; cudaMalloc(&o, 8); cudaMalloc(&c, 8);
  const int iters = 1000;
  unsigned long long h;
#define RUN(T) k_bar<T><<<1, T>>>(o, c, iters); k_bar<T><<<1, T>>>(o, c, iters); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("%4d threads: %.0f cycles per (load, barrier, store, barrier)\n", T, (double)h / iters);
  RUN(128) RUN(256) RUN(512) RUN(1024)
  return 0;
}
