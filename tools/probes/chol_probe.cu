// Standalone timing probe for k_chol_cluster phases (not part of the library).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#define CHOL_PROBE 1
__device__ unsigned long long g_t[64];
__device__ long long g_c[64];
__global__ void k_timer_res(unsigned long long* out) {
  unsigned long long prev, t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(prev));
  unsigned long long mind = ~0ull; int changes = 0; long long c0 = clock64();
  while (changes < 100) { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); if (t != prev) { if (t - prev < mind) mind = t - prev; prev = t; ++changes; } }
  out[0] = mind; out[1] = clock64() - c0;
}
#include "../../paper_2006_03970_b200/csrc/k_newton.cuh"
using namespace ssn;

__global__ void k_empty_cluster() {
  namespace cg = cooperative_groups;
  cg::this_cluster().sync();
}
__global__ void k_diag_only(double* M, int ld, int N, int* info, unsigned long long* t) {
  unsigned long long t0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  long long c0 = clock64();
  __shared__ double T[32 * 33 + kDiagScratch];  // diag tile + factor scratch
  if (threadIdx.x < 32) load_tile_rows(M, ld, 0, 0, N + 1, N, T, threadIdx.x);
  __syncthreads();
  if (threadIdx.x < 128) diag_factor4(T, M, ld, 0, N < 32 ? N : 32, N + 1 < 32 ? N + 1 : 32, M + (size_t)ld * N, nullptr, info, T + 32 * 33, threadIdx.x);
  __syncthreads();
  unsigned long long t1; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  long long c1 = clock64();
  if (threadIdx.x == 0) { t[0] = t1 - t0; t[1] = c1 - c0; }
}
// dependent DFMA chain of 10000 steps: cycles and ns
__global__ void k_chain(double* out, unsigned long long* t) {
  unsigned long long t0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  long long c0 = clock64();
  double x = threadIdx.x * 1e-3;
  for (int i = 0; i < 10000; ++i) x = fma(x, 0.999999, 1e-7);
  long long c1 = clock64();
  unsigned long long t1; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) { t[2] = t1 - t0; t[3] = c1 - c0; }
}

int main() {
  { unsigned long long* d; cudaMalloc(&d, 16); k_timer_res<<<1,1>>>(d); unsigned long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost); printf("globaltimer: min step %llu ns, 100 changes in %llu cycles\n", h[0], h[1]); }
  for (int N : {8, 32, 64, 200, 500}) {
    int ld = N + 1;
    std::vector<double> h((size_t)ld * N);
    srand(1);
    // SPD: identity * N + random small
    for (int j = 0; j < N; ++j) for (int i = 0; i < ld; ++i) h[i + (size_t)j * ld] = (i == j) ? N + 1.0 : ((i < N) ? 0.01 * ((i * 7 + j * 13) % 11) : 1.0);
    for (int j = 0; j < N; ++j) for (int i = 0; i < N; ++i) h[i + (size_t)j * ld] = h[(i > j ? i : j) + (size_t)(i > j ? j : i) * ld];
    double *dM, *dout, *dW, *dd; int* info; unsigned long long* dt;
    cudaMalloc(&dM, (h.size() + 4096) * 8); cudaMalloc(&dout, N * 8); cudaMalloc(&dW, 33 * 32 * 8 * ((N + 31) / 32)); cudaMalloc(&info, 4); cudaMalloc(&dt, 64 * 8); cudaMalloc(&dd, 8); int* kf; cudaMalloc(&kf, 1024); cudaMemset(kf, 0, 1024);
    size_t smem = kCholSmem;
    cudaFuncSetAttribute(k_chol_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_chol_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k_empty_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int cs : {1, 8, 16}) {
      cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(cs); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaMemcpy(dM, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
        cudaEventRecord(e0);
        cudaLaunchKernelEx(&cfg, k_chol_cluster, dM, N, N + 1, ld, dout, 1.0, (const double*)nullptr, (double*)nullptr, dW, info, (const double*)nullptr, (double*)nullptr, (const DirGeo*)nullptr, 0, kf, 0, (const CholArgs*)nullptr);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      printf("N=%4d cluster=%2d chol_cluster %8.1f us  err=%s\n", N, cs, best * 1e3, cudaGetErrorString(cudaGetLastError()));
      unsigned long long ts[64]; cudaMemcpyFromSymbol(ts, g_t, sizeof(ts));
      long long cs_[64]; cudaMemcpyFromSymbol(cs_, g_c, sizeof(cs_));
      printf("   cycles(k from start):");
      for (int q = 1; q < 60; ++q) if (ts[q] > ts[0] && ts[q] - ts[0] < 100000000ull) printf(" [%d]%.1f", q, (cs_[q] - cs_[0]) / 1000.0);
      printf("\n");
      printf("   stamps(us from start):");
      for (int q = 1; q < 60; ++q) if (ts[q] > ts[0] && ts[q] - ts[0] < 100000000ull) printf(" [%d]%.1f", q, (ts[q] - ts[0]) / 1000.0);
      printf("\n");
            { unsigned long long z[64] = {0}; cudaMemcpyToSymbol(g_t, z, sizeof(z)); }
      float bestE = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        cudaLaunchKernelEx(&cfg, k_empty_cluster);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < bestE) bestE = ms;
      }
      printf("           empty cluster kernel %8.1f us\n", bestE * 1e3);
    }
    cudaMemcpy(dM, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    k_diag_only<<<1, 256>>>(dM, ld, N, info, dt);
    k_chain<<<1, 32>>>(dout, dt);
    unsigned long long tt[4]; cudaMemcpy(tt, dt, 32, cudaMemcpyDeviceToHost);
    printf("           diag factor alone %8.2f us, %llu cycles -> %.0f MHz; fma chain 1e4: %.2f us %llu cycles (%.0f MHz, %.2f cyc/fma)\n", tt[0] / 1000.0, tt[1], tt[1] * 1000.0 / tt[0], tt[2] / 1000.0, tt[3], tt[3] * 1000.0 / tt[2], tt[3] / 1e4);
    cudaFree(dM); cudaFree(dout); cudaFree(dW); cudaFree(info); cudaFree(dt); cudaFree(dd);
  }
  return 0;
}
