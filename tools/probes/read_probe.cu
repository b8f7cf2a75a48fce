// Probe: the HBM READ ceiling on this B200, for the roofline of K1 (a read-dominated stream: 8mn bytes
// in, 8n out).  The driver's MEASURED_PEAKS hbm_gbs is a copy (read + write); K1 reads.  Streams a
// 40 GB buffer (cfg5's A) with
//   ldg  : grid-stride 16-byte loads (ld.global.nc.v2.f64), U independent loads in flight per thread,
//          grid = 148 × B CTAs of 256 threads;
//   bulk : one producer lane per CTA issuing cp.async.bulk of T-byte chunks into an S-stage shared ring
//          (K1's load path without its arithmetic), consumers only release the stage;
// and reports the best of R timed repetitions (CUDA events) per variant, in GB/s of bytes read.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_ldg(const double2* __restrict__ p, int64_t n2, double* sink) {
  constexpr int U = 8;
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n2; i += U * stride) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldg(p + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y;
  }
  for (; i < n2; i += stride) acc += p[i].x + p[i].y;
  if (acc == 12345.678) *sink = acc;
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// contiguous chunk range per CTA (as K1's tile ranges), S-stage ring, warp 0 lane 0 = producer,
// warps 1..7 take stages round-robin and release them after touching one word
__global__ void k_bulk(const char* __restrict__ p, int64_t nchunks, int chunk, int S, int pieces, double* sink) {
  extern __shared__ __align__(128) char smem[];
  uint64_t* full = (uint64_t*)smem;
  uint64_t* empty = full + 32;  // ≤ 32 stages
  char* ring = smem + 512;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t c0 = nchunks * blockIdx.x / gridDim.x, c1 = nchunks * (blockIdx.x + 1) / gridDim.x;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(full + s)));
      asm volatile("mbarrier.init.shared.b64 [%0], 7;" ::"r"(su32(empty + s)));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  double acc = 0.0;
  if (warp == 0) {
    if (lane == 0)
      for (int64_t c = c0; c < c1; ++c) {
        const int it = (int)(c - c0), s = it % S;
        if (it >= S) {  // wait until the consumers released this stage
          const uint32_t par = ((it / S) - 1) & 1;
          asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared.b64 P, [%0], %1;\n@!P bra W;\n}" ::"r"(
                           su32(empty + s)),
                       "r"(par));
        }
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(full + s)), "r"(chunk));
        const int pb = chunk / pieces;  // one stage issued as `pieces` bulk copies on the same barrier
        for (int q = 0; q < pieces; ++q)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  su32(ring + (size_t)s * chunk + q * pb)),
              "l"(p + c * (int64_t)chunk + q * pb), "r"(pb), "r"(su32(full + s))
              : "memory");
      }
  } else {
    for (int64_t c = c0; c < c1; ++c) {
      const int it = (int)(c - c0), s = it % S;
      const uint32_t par = (it / S) & 1;
      asm volatile("{\n.reg .pred P;\nW2: mbarrier.try_wait.parity.shared.b64 P, [%0], %1;\n@!P bra W2;\n}" ::"r"(
                       su32(full + s)),
                   "r"(par));
      if (lane == 0) acc += *(const double*)(ring + (size_t)s * chunk + 8 * warp);
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(su32(empty + s)));
    }
  }
  if (acc == 12345.678) *sink = acc;
}

int main(int argc, char** argv) {
  const int64_t bytes = (argc > 1 ? atoll(argv[1]) : 40000000000LL) / 4096 * 4096;
  const int R = 5;
  char* p;
  double* sink;
  if (cudaMalloc(&p, bytes) != cudaSuccess) {
    printf("alloc failed\n");
    return 1;
  }
  cudaMemset(p, 1, bytes);
  cudaMalloc(&sink, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  auto timeit = [&](auto launch) {
    float best = 1e30f;
    launch();
    cudaDeviceSynchronize();
    for (int r = 0; r < R; ++r) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    return best;
  };
  for (int B : {1, 2, 4, 8}) {
    const float ms = timeit([&] { k_ldg<<<nsm * B, 256>>>((const double2*)p, bytes / 16, sink); });
    printf("{\"variant\": \"ldg\", \"ctas_per_sm\": %d, \"ms\": %.3f, \"GBps\": %.1f}\n", B, ms, bytes / ms / 1e6);
  }
  struct Cfg { int chunk, S, pieces; };
  const Cfg cfgs[] = {{32768, 6, 1}, {32768, 6, 2}, {32768, 6, 4}, {32768, 4, 2}, {32000, 6, 1}, {32000, 6, 2},
                      {16384, 6, 1}, {16384, 8, 1}, {16384, 12, 1}, {16384, 12, 2}, {8192, 12, 1}, {8192, 24, 1},
                      {65536, 3, 4}, {4096, 32, 1}};
  for (const Cfg& c : cfgs) {
    const int smem = 512 + c.S * c.chunk;
    if (smem > 227 * 1024 || c.S > 32) continue;
    cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int64_t nch = bytes / c.chunk;
    const float ms = timeit([&] { k_bulk<<<nsm, 256, smem>>>(p, nch, c.chunk, c.S, c.pieces, sink); });
    printf("{\"variant\": \"bulk\", \"chunk\": %d, \"stages\": %d, \"pieces\": %d, \"ms\": %.3f, \"GBps\": %.1f}\n",
           c.chunk, c.S, c.pieces, ms, (double)nch * c.chunk / ms / 1e6);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error: %s\n", cudaGetErrorString(e));
  return 0;
}
