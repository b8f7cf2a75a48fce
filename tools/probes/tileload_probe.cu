// Probe: the K4 worker load pattern in isolation — 15 (or 148) CTAs × 8 warps, each thread issuing
// the 24 loads of one trailing-update job (8 rows × 8 columns of two 32 × 32 tiles and an 8-value
// accumulator fragment) from a 2 MB column-major matrix (ld = 501), N rounds; reports µs per round
// for __ldcg (L2) and __ldg (L1-cacheable), plus the same with the matrix freshly written by other
// CTAs (write, grid barrier via a second kernel, read).
#include <cstdio>
__global__ void k_rounds(const double* M, int ld, int ntiles, int rounds, int mode, double* sink) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, qw = warp & 3, g = lane >> 2, t = lane & 3;
  double s = 0.0;
  for (int rd = 0; rd < rounds; ++rd) {
    const int job = (blockIdx.x * 2 + (warp >> 2) + rd * 37) % (ntiles * ntiles);
    const int i0 = (job / ntiles) * 32, j0 = (job % ntiles) * 32, k0 = ((rd * 7) % ntiles) * 32;
    double v[24];
    if (mode < 2) {  // K4 v4 pattern: lane (g, t) → row 8qw + g, columns 8t + e
      const double* sa = M + (int64_t)(k0 + 8 * t) * ld + i0 + 8 * qw + g;
      const double* sb = M + (int64_t)(k0 + 8 * t) * ld + j0 + 8 * qw + g;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        v[e] = mode ? __ldg(sa + e * ld) : __ldcg(sa + e * ld);
        v[8 + e] = mode ? __ldg(sb + e * ld) : __ldcg(sb + e * ld);
        v[16 + e] = mode ? __ldg(M + (int64_t)(j0 + e) * ld + i0 + lane) : __ldcg(M + (int64_t)(j0 + e) * ld + i0 + lane);
      }
    } else {  // coalesced: lane = row, warp qw takes columns 8qw .. 8qw+7 of each tile
      const double* sa = M + (int64_t)(k0 + 8 * qw) * ld + i0 + lane;
      const double* sb = M + (int64_t)(k0 + 8 * qw) * ld + j0 + lane;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        v[e] = __ldcg(sa + e * ld);
        v[8 + e] = __ldcg(sb + e * ld);
        v[16 + e] = __ldcg(M + (int64_t)(j0 + 8 * qw + e) * ld + i0 + lane);
      }
    }
#pragma unroll
    for (int e = 0; e < 24; ++e) s += v[e];
    __syncthreads();
  }
  if (s == 12345.678) sink[0] = s;
}
int main() {
  const int N = 500, ld = 501, ntiles = 15;
  double* M; cudaMalloc(&M, (size_t)ld * N * 8 + 4096);
  cudaMemset(M, 0, (size_t)ld * N * 8);
  double* sink; cudaMalloc(&sink, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int grid : {15, 148})
    for (int mode : {0, 1, 2}) {
      const int rounds = 200;
      k_rounds<<<grid, 256>>>(M, ld, ntiles, 10, mode, sink);
      cudaEventRecord(e0);
      k_rounds<<<grid, 256>>>(M, ld, ntiles, rounds, mode, sink);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("grid %3d %s: %.2f us per round (24 loads/thread + syncthreads)\n", grid, mode == 2 ? "coalesced ldcg" : (mode ? "ldg " : "ldcg"), ms * 1e3 / rounds);
    }
  return 0;
}
