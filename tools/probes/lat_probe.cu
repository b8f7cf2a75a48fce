#include <cstdio>
__global__ void k(double* out, long long* cyc, double seed) {
  double x = seed + threadIdx.x * 1e-9;
  long long c0 = clock64();
  for (int i = 0; i < 1000; ++i) x = sqrt(x) + 1.0;
  long long c1 = clock64();
  for (int i = 0; i < 1000; ++i) x = 1.0 / x + 1.0;
  long long c2 = clock64();
  for (int i = 0; i < 1000; ++i) x = rsqrt(x) + 1.0;
  long long c3 = clock64();
  for (int i = 0; i < 1000; ++i) x = __drcp_rn(x) + 1.0;
  long long c4 = clock64();
  for (int i = 0; i < 1000; ++i) x = __dsqrt_rn(x) + 1.0;
  long long c5 = clock64();
  double y = x;
  for (int i = 0; i < 1000; ++i) y = __fma_rn(y, 0.999, 1e-3);
  long long c6 = clock64();
  out[threadIdx.x] = x + y;
  if (threadIdx.x == 0) { cyc[0] = c1 - c0; cyc[1] = c2 - c1; cyc[2] = c3 - c2; cyc[3] = c4 - c3; cyc[4] = c5 - c4; cyc[5] = c6 - c5; }
}
__global__ void k_bar(long long* cyc) {
  __shared__ double s[256];
  long long c0 = clock64();
  for (int i = 0; i < 1000; ++i) { s[threadIdx.x] = i; __syncthreads(); }
  long long c1 = clock64();
  for (int i = 0; i < 1000; ++i) { asm volatile("bar.sync 2, 128;" ::: "memory"); }
  long long c2 = clock64();
  for (int i = 0; i < 1000; ++i) { __syncwarp(); }
  long long c3 = clock64();
  if (threadIdx.x == 0) { cyc[0] = c1 - c0; cyc[1] = c2 - c1; cyc[2] = c3 - c2; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 64);
  for (int rep = 0; rep < 2; ++rep) {
    k<<<1, 32>>>(o, c, 2.0);
    long long h[6]; cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
    printf("per-op latency (cycles, chain of 1000): sqrt %.1f  1/x %.1f  rsqrt %.1f  drcp_rn %.1f  dsqrt_rn %.1f  fma %.1f\n", h[0] / 1e3, h[1] / 1e3, h[2] / 1e3, h[3] / 1e3, h[4] / 1e3, h[5] / 1e3);
  }
  k_bar<<<1, 128>>>(c);
  long long h[3]; cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
  printf("syncthreads(128) %.1f  bar.sync named %.1f  syncwarp %.1f cycles\n", h[0] / 1e3, h[1] / 1e3, h[2] / 1e3);
  return 0;
}
