// Probe: cluster barrier latency (16-CTA and 8-CTA clusters), dependent L2 load latency, and
// bar.sync latency — the primitives that bound the per-panel critical path of K4.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k_clsync(int iters, unsigned long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  long long c0 = clock64();
  for (int i = 0; i < iters; ++i) cl.sync();
  long long c1 = clock64();
  if (threadIdx.x == 0 && cl.block_rank() == 0) out[0] = c1 - c0;
}
__global__ void k_clsync_split(int iters, unsigned long long* out) {  // arrive.release / wait.acquire
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  long long c0 = clock64();
  for (int i = 0; i < iters; ++i) {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  long long c1 = clock64();
  if (threadIdx.x == 0 && cl.block_rank() == 0) out[1] = c1 - c0;
}
__global__ void k_barsync(int iters, unsigned long long* out) {
  long long c0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  long long c1 = clock64();
  if (threadIdx.x == 0) out[2] = c1 - c0;
}
__global__ void k_chase(const long long* p, int iters, unsigned long long* out, long long* sink) {
  long long j = 0;
  long long c0 = clock64();
  for (int i = 0; i < iters; ++i) j = __ldcg(p + j);
  long long c1 = clock64();
  *sink = j;
  out[3] = c1 - c0;
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 64);
  long long* p; cudaMalloc(&p, (1 << 20) * 8);
  long long* sink; cudaMalloc(&sink, 8);
  long long* h = new long long[1 << 20];
  for (int i = 0; i < (1 << 20); ++i) h[i] = (i * 7919 + 4099) % (1 << 20);
  cudaMemcpy(p, h, (1 << 20) * 8, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_clsync, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_clsync_split, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {2, 8, 16}) {
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(cs); cfg.blockDim = dim3(256);
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_clsync, 1000, d);
    cudaLaunchKernelEx(&cfg, k_clsync_split, 1000, d);
    cudaDeviceSynchronize();
    unsigned long long o[4]; cudaMemcpy(o, d, 32, cudaMemcpyDeviceToHost);
    printf("cluster %2d: cl.sync %.0f cyc, arrive.release+wait.acquire %.0f cyc  (%s)\n", cs, o[0] / 1000.0, o[1] / 1000.0, cudaGetErrorString(cudaGetLastError()));
  }
  k_barsync<<<1, 256>>>(1000, d);
  k_chase<<<1, 1>>>(p, 2000, d, sink);  // warm
  k_chase<<<1, 1>>>(p, 2000, d, sink);
  cudaDeviceSynchronize();
  unsigned long long o[4]; cudaMemcpy(o, d, 32, cudaMemcpyDeviceToHost);
  printf("__syncthreads(256) %.0f cyc; dependent L2 load (ld.cg) %.0f cyc\n", o[2] / 1000.0, o[3] / 2000.0);
  return 0;
}
