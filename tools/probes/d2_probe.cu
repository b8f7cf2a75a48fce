// Probe (not part of the library): k_chol_d2 (split-ownership DSMEM Cholesky) vs k_chol_dsm and a
// host fp64 Cholesky solve on random SPD systems M = I + G Gᵀ/N (ld = N + 1, rhs in row N), with
// per-call timing of both kernels.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>
#define D2_PROBE 1
#include "../../paper_2006_03970_b200/csrc/k_chol_d2.cuh"
using namespace ssn;

static void host_solve(const std::vector<double>& Mh, int N, int ld, std::vector<double>& x) {
  std::vector<double> L((size_t)N * N, 0.0);
  for (int j = 0; j < N; ++j) {
    double d = Mh[j + (size_t)j * ld];
    for (int p = 0; p < j; ++p) d -= L[j + (size_t)p * N] * L[j + (size_t)p * N];
    d = std::sqrt(d);
    L[j + (size_t)j * N] = d;
    for (int i = j + 1; i < N; ++i) {
      double s = Mh[i + (size_t)j * ld];
      for (int p = 0; p < j; ++p) s -= L[i + (size_t)p * N] * L[j + (size_t)p * N];
      L[i + (size_t)j * N] = s / d;
    }
  }
  std::vector<double> z(N);
  for (int i = 0; i < N; ++i) {  // rhs = row N: M[N + c·ld]
    double s = Mh[N + (size_t)i * ld];
    for (int p = 0; p < i; ++p) s -= L[i + (size_t)p * N] * z[p];
    z[i] = s / L[i + (size_t)i * N];
  }
  x.assign(N, 0.0);
  for (int i = N - 1; i >= 0; --i) {
    double s = z[i];
    for (int p = i + 1; p < N; ++p) s -= L[p + (size_t)i * N] * x[p];
    x[i] = s / L[i + (size_t)i * N];
  }
}

int main(int argc, char** argv) {
  for (auto kf : {k_chol_d2t<4>, k_chol_d2t<5>}) {  // (6 chain CTAs needs kD2Slots = 13)  // kD2Slots must cover 6 (13 slots) for this probe
    cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kD2Smem);
    cudaFuncSetAttribute(kf, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  }
  cudaFuncSetAttribute(k_chol_dsm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDsmSmem);
  cudaFuncSetAttribute(k_chol_dsm, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  std::vector<int> Ns = {161, 192, 200, 255, 256, 257, 300, 391, 435, 480, 500, 511, 512};
  if (argc > 1) { Ns.clear(); for (int a = 1; a < argc; ++a) Ns.push_back(atoi(argv[a])); }
  printf("smem d2 %zu dsm %zu\n", kD2Smem, kDsmSmem);
  std::mt19937_64 rng(7);
  std::normal_distribution<double> nd;
  int fails = 0;
  for (int N : Ns) {
    const int ld = N + 1;
    std::vector<double> G((size_t)N * 2 * N);
    for (auto& v : G) v = nd(rng);
    std::vector<double> h((size_t)ld * N, 0.0);
    for (int j = 0; j < N; ++j)
      for (int i = j; i < N; ++i) {
        double s = 0.0;
        for (int p = 0; p < 2 * N; ++p) s += G[i + (size_t)p * N] * G[j + (size_t)p * N];
        s /= N;
        if (i == j) s += 1.0;
        h[i + (size_t)j * ld] = s;
        h[j + (size_t)i * ld] = s;
      }
    for (int c = 0; c < N; ++c) h[N + (size_t)c * ld] = nd(rng);
    std::vector<double> xr;
    host_solve(h, N, ld, xr);
    double *dM, *dout, *dout2, *dot; int* info;
    cudaMalloc(&dM, h.size() * 8); cudaMalloc(&dout, N * 8); cudaMalloc(&dout2, N * 8); cudaMalloc(&info, 4);
    cudaMalloc(&dot, 8);
    cudaMemset(info, 0, 4);
    cudaMemcpy(dM, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kDsmCS); cfg.blockDim = dim3(256);
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kDsmCS; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    const DirGeo* nog = nullptr;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float msv[2] = {0, 0};
    double ev[2] = {0, 0};
    int iv[2] = {0, 0};
    cudaError_t err = cudaSuccess;
    double xm = 0;
    for (int pass = 0; pass < 2; ++pass)
      for (int v = 0; v < 2; ++v) {  // chain CTAs: 4 (round-2 design), 5 (the library's kD2Chain)
        auto kf = v == 0 ? k_chol_d2t<4> : k_chol_d2t<5>;
        cfg.dynamicSmemBytes = kD2Smem;
        cudaMemset(info, 0, 4);
        for (int it = 0; it < 3; ++it)
          cudaLaunchKernelEx(&cfg, kf, (const double*)dM, N, ld, dout, 1.0, (const double*)nullptr, (double*)nullptr,
                             info, (const double*)nullptr, (double*)nullptr, nog, 0, 0, kDsmMaxN,
                             (const CholArgs*)nullptr);
        cudaEventRecord(e0);
        for (int it = 0; it < 20; ++it)
          cudaLaunchKernelEx(&cfg, kf, (const double*)dM, N, ld, dout, 1.0, (const double*)nullptr, (double*)nullptr,
                             info, (const double*)nullptr, (double*)nullptr, nog, 0, 0, kDsmMaxN,
                             (const CholArgs*)nullptr);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&msv[v], e0, e1);
        err = cudaDeviceSynchronize();
        if (err != cudaSuccess) break;
        std::vector<double> x2(N);
        cudaMemcpy(x2.data(), dout, N * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(&iv[v], info, 4, cudaMemcpyDeviceToHost);
        double e2 = 0;
        xm = 0;
        for (int i = 0; i < N; ++i) {
          xm = fmax(xm, fabs(xr[i]));
          e2 = fmax(e2, fabs(x2[i] - xr[i]));
        }
        ev[v] = e2;
      }
    bool ok = err == cudaSuccess;
    for (int v = 0; v < 2; ++v) ok = ok && iv[v] == 0 && ev[v] <= 1e-11 * xm;
    fails += !ok;
    printf("N=%3d chain4 %6.1f us  chain5 %6.1f us  err %.2e %.2e %s %s\n", N, msv[0] * 1e3 / 20, msv[1] * 1e3 / 20,
           ev[0] / xm, ev[1] / xm, cudaGetErrorString(err), ok ? "OK" : "FAIL");
    if (getenv("D2_TIMELINE")) {
      unsigned long long tl[18][12];
      cudaMemcpyFromSymbol(tl, g_d2, sizeof(tl));
      const unsigned long long t0 = tl[17][0];
      auto f = [&](unsigned long long v) { return v >= t0 && v - t0 < 10000000ull ? (v - t0) * 1e-3 : -1.0; };
      printf("  start→factor-loop-end %.1f  end %.1f us\n", f(tl[17][1]), f(tl[17][2]));
      printf("   j:  fac0  facdone  W_j  q1start q1strip q1push L(j+1,j)  v_j | h(j+2,j): Astart Adone Wgot publish\n");
      for (int j = 0; j < (N + 31) / 32; ++j) {
        printf("  %2d: %6.1f %6.1f %6.1f %6.1f %6.1f %6.1f %6.1f %6.1f\n", j, f(tl[j][0]), f(tl[j][3]), f(tl[j][1]), f(tl[j][4]), f(tl[j][6]), f(tl[j][7]), f(tl[j][2]), f(tl[j][5]));
        printf("      %6.1f %6.1f %6.1f %6.1f\n", f(tl[j][10]), f(tl[j][11]), f(tl[j][9]), f(tl[j][8]));
      }
    }
    cudaFree(dM); cudaFree(dout); cudaFree(dout2); cudaFree(info); cudaFree(dot);
  }
  printf("fails %d\n", fails);
  return fails != 0;
}
