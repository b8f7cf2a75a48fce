// Probe: the library's diag_factor4 (one 32 × 32 diagonal tile, 4 warps), cycles end to end,
// and the accuracy of L Lᵀ = A and W L = I.
#include <cstdio>
#include <cmath>
#include "../../paper_2006_03970_b200/csrc/k_newton.cuh"
using namespace ssn;
__global__ void k_d4(const double* Sg, double* M, double* W, int* info, unsigned long long* cyc) {
  __shared__ double S[CHT * TLD + kDiagScratch];
  for (int e = threadIdx.x; e < CHT * TLD; e += 128) S[e] = Sg[e];
  __syncthreads();
  long long c0 = clock64();
  diag_factor4(S, M, 32, 0, 32, 32, W, nullptr, info, S + CHT * TLD, threadIdx.x);
  long long c1 = clock64();
  if (threadIdx.x == 0) cyc[0] = c1 - c0;
}
int main() {
  double h[CHT * TLD];
  for (int r = 0; r < CHT; ++r)
    for (int c = 0; c < TLD; ++c) h[r * TLD + c] = (r == c) ? 4.0 + r : ((c < CHT) ? 0.3 * sin(r * 7.0 + c * 13.0 + (r > c ? r * c : c * r)) : 0.0);
  for (int r = 0; r < CHT; ++r) for (int c = 0; c < r; ++c) h[c * TLD + r] = h[r * TLD + c];
  double *dS, *dM, *dW; int* info; unsigned long long* cyc;
  cudaMalloc(&dS, sizeof(h)); cudaMalloc(&dM, 32 * 32 * 8); cudaMalloc(&dW, 32 * 32 * 8); cudaMalloc(&info, 4); cudaMalloc(&cyc, 64);
  cudaMemcpy(dS, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaMemset(dM, 0, 32 * 32 * 8); cudaMemset(info, 0, 4);
  for (int rep = 0; rep < 3; ++rep) k_d4<<<1, 128>>>(dS, dM, dW, info, cyc);
  cudaDeviceSynchronize();
  unsigned long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  double L[32 * 32], W[32 * 32]; int inf;
  cudaMemcpy(L, dM, sizeof(L), cudaMemcpyDeviceToHost); cudaMemcpy(W, dW, sizeof(W), cudaMemcpyDeviceToHost);
  cudaMemcpy(&inf, info, 4, cudaMemcpyDeviceToHost);
  double e1 = 0, e2 = 0;
  for (int i = 0; i < 32; ++i) for (int j = 0; j <= i; ++j) {
    double s = 0; for (int p = 0; p <= j; ++p) s += L[i + p * 32] * L[j + p * 32];
    e1 = fmax(e1, fabs(s - h[i * TLD + j]));
    double t = 0; for (int p = j; p <= i; ++p) t += W[i * 32 + p] * L[p + j * 32];
    e2 = fmax(e2, fabs(t - (i == j)));
  }
  printf("diag_factor4: %llu cycles (%.0f per pivot)  |LL'-A|max %.2e  |WL-I|max %.2e  info %d  %s\n", c, c / 32.0, e1, e2, inf,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
