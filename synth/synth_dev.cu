/*
 * synth/synth_dev.cu — device side of the seeded input generator (gen_core.h).
 * Writes the SAME bytes as synth_host.c's synth_fill_A directly into device
 * memory so that 40 GB designs never cross PCIe.  Built with nvcc
 * --fmad=false; gen_core.h uses __d*_rn intrinsics on the device.
 * No SsNAL-EN arithmetic lives here.
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include "gen_core.h"

/* One thread per column: the raw column is regenerated in each of the three
 * standardisation passes (sum; centred sum of squares; write), reproducing
 * sx_standardise's exact operation order without storing the raw values. */
template <int KIND>
__global__ void k_gen_columns(uint64_t seed, int64_t m, int64_t n, int64_t j0, int64_t j1, double* out,
                              int* bad) {
  int64_t j = j0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= j1) return;
  auto raw = [&](int64_t k) -> double {
    if (KIND == SX_GENO_STD) return sx_geno_entry(seed, m, n, k, j);
    return sx_iid_entry(seed, m, k, j);
  };
  double s = 0.0;
  for (int64_t k = 0; k < m; ++k) s = SX_ADD(s, raw(k));
  double mean = SX_DIV(s, (double)m);
  double ss = 0.0;
  for (int64_t k = 0; k < m; ++k) {
    double c = SX_SUB(raw(k), mean);
    ss = SX_ADD(ss, SX_MUL(c, c));
  }
  double* col = out + (j - j0) * m;
  if (!(ss > 0.0)) {
    atomicAdd(bad, 1);
    for (int64_t k = 0; k < m; ++k) col[k] = SX_SUB(raw(k), mean);
    return;
  }
  double nrm = (KIND == SX_IID_UNIT_L2) ? SX_SQRT(ss) : SX_SQRT(SX_DIV(ss, (double)m));
  for (int64_t k = 0; k < m; ++k) col[k] = SX_DIV(SX_SUB(raw(k), mean), nrm);
}

/* AR(1): one thread per (row k, chunk c); raw values written coalesced. */
__global__ void k_gen_ar1_raw(uint64_t seed, int64_t m, int64_t n, int64_t j0, int64_t j1, double* out) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t c = blockIdx.y + (int64_t)blockIdx.z * 65535;
  if (k >= m) return;
  int64_t c0 = (j0 / SX_AR1_CHUNK + c) * SX_AR1_CHUNK;
  if (c0 >= j1) return;
  int64_t ce = c0 + SX_AR1_CHUNK < n ? c0 + SX_AR1_CHUNK : n;
  double a = sx_ar1_start(seed, m, k, c0);
  for (int64_t j = c0; j < ce; ++j) {
    if (j > c0) a = sx_ar1_step(a, sx_iid_entry(seed, m, k, j));
    if (j >= j0 && j < j1) out[(j - j0) * m + k] = a;
  }
}

__global__ void k_standardise(int64_t m, int64_t ncols, double* out, int* bad) {
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= ncols) return;
  if (!sx_standardise(out + j * m, m, 0)) atomicAdd(bad, 1);
}

/* Packed genotype codes, one thread per column (gen_core.h sx_geno_packed). */
__global__ void k_gen_geno_packed(uint64_t seed, int64_t m, int64_t n, int64_t j0, int64_t j1, uint8_t* codes,
                                  int64_t stride, double* tab, int* bad) {
  int64_t j = j0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= j1) return;
  if (!sx_geno_packed(seed, m, n, j, codes + (j - j0) * stride, stride, tab + (j - j0) * 3)) atomicAdd(bad, 1);
}

extern "C" {

/* Same contract as synth_fill_A (host) but out is a device pointer.
 * Returns 0 / number of zero-variance columns / -1 bad args / -2 CUDA error. */
int synth_fill_A_device(int kind, uint64_t seed, int64_t m, int64_t n, int64_t j0, int64_t j1, double* out,
                        void* stream) {
  if (m < 1 || n < 1 || j0 < 0 || j1 > n || j0 > j1) return -1;
  if (j1 == j0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  int* dbad = nullptr;
  if (cudaMallocAsync((void**)&dbad, sizeof(int), st) != cudaSuccess) return -2;
  cudaMemsetAsync(dbad, 0, sizeof(int), st);
  int64_t ncols = j1 - j0;
  const int T = 128;
  unsigned nb = (unsigned)((ncols + T - 1) / T);
  switch (kind) {
    case SX_IID_UNIT_L2: k_gen_columns<SX_IID_UNIT_L2><<<nb, T, 0, st>>>(seed, m, n, j0, j1, out, dbad); break;
    case SX_IID_STD: k_gen_columns<SX_IID_STD><<<nb, T, 0, st>>>(seed, m, n, j0, j1, out, dbad); break;
    case SX_GENO_STD: k_gen_columns<SX_GENO_STD><<<nb, T, 0, st>>>(seed, m, n, j0, j1, out, dbad); break;
    case SX_AR1_STD: {
      int64_t nch = (j1 - 1) / SX_AR1_CHUNK - j0 / SX_AR1_CHUNK + 1;
      dim3 g((unsigned)((m + T - 1) / T), (unsigned)(nch < 65535 ? nch : 65535), (unsigned)((nch + 65534) / 65535));
      k_gen_ar1_raw<<<g, T, 0, st>>>(seed, m, n, j0, j1, out);
      k_standardise<<<nb, T, 0, st>>>(m, ncols, out, dbad);
      break;
    }
    default: cudaFreeAsync(dbad, st); return -1;
  }
  int hbad = 0;
  cudaMemcpyAsync(&hbad, dbad, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(dbad, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return -2;
  if (cudaGetLastError() != cudaSuccess) return -2;
  return hbad;
}

/* Device twin of synth_geno_codes (codes, tab are device pointers). */
int synth_geno_codes_device(uint64_t seed, int64_t m, int64_t n, int64_t j0, int64_t j1, uint8_t* codes,
                            int64_t stride, double* tab, void* stream) {
  if (m < 1 || n < 1 || j0 < 0 || j1 > n || j0 > j1 || stride < (m + 3) / 4) return -1;
  if (j1 == j0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  int* dbad = nullptr;
  if (cudaMallocAsync((void**)&dbad, sizeof(int), st) != cudaSuccess) return -2;
  cudaMemsetAsync(dbad, 0, sizeof(int), st);
  const int T = 128;
  k_gen_geno_packed<<<(unsigned)((j1 - j0 + T - 1) / T), T, 0, st>>>(seed, m, n, j0, j1, codes, stride, tab, dbad);
  int hbad = 0;
  cudaMemcpyAsync(&hbad, dbad, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(dbad, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return -2;
  if (cudaGetLastError() != cudaSuccess) return -2;
  return hbad;
}

}  // extern "C"
