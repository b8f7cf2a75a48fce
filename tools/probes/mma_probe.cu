// Probe: FP64 throughput per warp / per SM — DMMA m8n8k4 tile products (as in K4's tile_mma)
// versus scalar DFMA, with 1, 2, 4 and 8 warps per CTA.
#include <cstdio>
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
__global__ void k_dmma(int iters, double* out, unsigned long long* cyc) {
  double acc[4][4][2] = {};
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  long long c0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int rb = 0; rb < 4; ++rb)
#pragma unroll
      for (int cb = 0; cb < 4; ++cb) dmma(acc[rb][cb], a, b);
  }
  long long c1 = clock64();
  double s = 0;
  for (int rb = 0; rb < 4; ++rb) for (int cb = 0; cb < 4; ++cb) s += acc[rb][cb][0] + acc[rb][cb][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
}
__global__ void k_dfma(int iters, double* out, unsigned long long* cyc) {
  double acc[16];
  for (int j = 0; j < 16; ++j) acc[j] = threadIdx.x + j;
  const double a = 0.999999, b = 1e-7;
  long long c0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = fma(acc[j], a, b);
  }
  long long c1 = clock64();
  double s = 0;
  for (int j = 0; j < 16; ++j) s += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
}
int main() {
  double* o; cudaMalloc(&o, 1 << 20);
  unsigned long long* c; cudaMalloc(&c, 1024);
  const int it = 1000;
  for (int w : {1, 2, 4, 8}) {
    unsigned long long h;
    k_dmma<<<1, 32 * w>>>(it, o, c); cudaDeviceSynchronize();
    k_dmma<<<1, 32 * w>>>(it, o, c); cudaDeviceSynchronize();
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    const double fma_per_cyc = (double)w * it * 16 * 256 / h;
    k_dfma<<<1, 32 * w>>>(it, o, c); cudaDeviceSynchronize();
    unsigned long long h2; cudaMemcpy(&h2, c, 8, cudaMemcpyDeviceToHost);
    const double f2 = (double)w * it * 16 * 32 / h2;
    printf("warps %d: DMMA %.1f cyc/instr/warp -> %.1f FMA/clk/SM; DFMA %.2f cyc/instr/warp -> %.1f FMA/clk/SM\n", w,
           (double)h / (it * 16), fma_per_cyc, (double)h2 / (it * 16), f2);
  }
  return 0;
}
