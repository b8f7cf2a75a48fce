// Timeline probe for k_chol_dsm (not part of the library): per-CTA globaltimer stamps.
#include <cstdio>
#include <cstdlib>
#include <vector>
#define DSM_PROBE 1
#include "../../paper_2006_03970_b200/csrc/k_chol_dsm.cuh"
using namespace ssn;
int main() {
  cudaFuncSetAttribute(k_chol_dsm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDsmSmem);
  cudaFuncSetAttribute(k_chol_dsm, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int N : {100, 435, 500}) {
    int ld = N + 1;
    std::vector<double> h((size_t)ld * N);
    for (int j = 0; j < N; ++j)
      for (int i = 0; i < ld; ++i)
        h[i + (size_t)j * ld] = (i == j) ? N + 1.0 : ((i < N) ? 0.01 * (((i > j ? i : j) * 7 + (i > j ? j : i) * 13) % 11) : 1.0);
    double *dM, *dout; int* info;
    cudaMalloc(&dM, h.size() * 8); cudaMalloc(&dout, N * 8); cudaMalloc(&info, 4); cudaMemset(info, 0, 4);
    cudaMemcpy(dM, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kDsmCS); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = kDsmSmem;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kDsmCS; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const DirGeo* nog = nullptr;
    for (int it = 0; it < 3; ++it) cudaLaunchKernelEx(&cfg, k_chol_dsm, (const double*)dM, N, ld, dout, 1.0, (const double*)nullptr, (double*)nullptr, info, (const double*)nullptr, (double*)nullptr, nog, 0, kDsmMaxN, (const CholArgs*)nullptr);
    cudaEventRecord(e0);
    for (int it = 0; it < 20; ++it) cudaLaunchKernelEx(&cfg, k_chol_dsm, (const double*)dM, N, ld, dout, 1.0, (const double*)nullptr, (double*)nullptr, info, (const double*)nullptr, (double*)nullptr, nog, 0, kDsmMaxN, (const CholArgs*)nullptr);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("N=%d: %.1f us per call (%s)\n", N, ms * 1e3 / 20, cudaGetErrorString(cudaGetLastError()));
    unsigned long long t[kDsmCS][16];
    cudaMemcpyFromSymbol(t, g_dsm, sizeof(t));
    unsigned long long t0 = ~0ull;
    for (int j = 0; j < kDsmCS; ++j) if (t[j][0] && t[j][0] < t0) t0 = t[j][0];
    printf("  j: start  sync | diagabs  q1abs  factor  pub1  q0done q1done  vpub   end   (us from first start)\n");
    const int ntc = (N + 31) / 32;
    for (int j = 0; j < ntc; ++j) {
      auto f = [&](int i) { return t[j][i] >= t0 ? (t[j][i] - t0) * 1e-3 : -1.0; };
      printf("  %2d: %5.1f %5.1f | %6.1f %6.1f %6.1f %6.1f %6.1f %6.1f %6.1f %6.1f\n", j, f(0), f(1), f(2), f(8), f(3), f(4), f(5), f(9), f(6), f(7));
    }
    cudaFree(dM); cudaFree(dout); cudaFree(info);
  }
  return 0;
}
