// Probe: dependent-latency of FP64 ops on sm_100a (cycles per op, one warp).
#include <cstdio>
__global__ void k(double* out, long long* cyc, double seed) {
  double x = seed + threadIdx.x * 1e-9;
  long long c0 = clock64();
  for (int i = 0; i < 1000; ++i) x = fma(x, 0.9999999, 1e-9);
  long long c1 = clock64();
  for (int i = 0; i < 1000; ++i) x = x * 1.0000001;
  long long c2 = clock64();
  for (int i = 0; i < 1000; ++i) { double y; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); x = y; }
  long long c3 = clock64();
  for (int i = 0; i < 1000; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
  long long c4 = clock64();
  float f = (float)x;
  for (int i = 0; i < 1000; ++i) f = fmaf(f, 0.9999999f, 1e-9f);
  long long c5 = clock64();
  for (int i = 0; i < 1000; ++i) { float y; asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(f)); f = y; }
  long long c6 = clock64();
  out[threadIdx.x] = x + f;
  if (threadIdx.x == 0) { cyc[0] = c1 - c0; cyc[1] = c2 - c1; cyc[2] = c3 - c2; cyc[3] = c4 - c3; cyc[4] = c5 - c4; cyc[5] = c6 - c5; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 32 * 8); cudaMalloc(&c, 64);
  for (int r = 0; r < 2; ++r) k<<<1, 32>>>(o, c, 1.5);
  long long h[6]; cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
  printf("cycles/op: DFMA %.1f DMUL %.1f MUFU.rsqrt64 %.1f SHFL %.1f FFMA %.1f MUFU.rsqrt32 %.1f\n", h[0] / 1e3, h[1] / 1e3, h[2] / 1e3, h[3] / 1e3, h[4] / 1e3, h[5] / 1e3);
  return 0;
}
