// Probe: a cooperative (grid.sync) kernel launched with cudaLaunchKernelEx + the cooperative
// attribute, captured into the body of a conditional WHILE node; grid.sync latency at 148 CTAs.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k_coop(int* cnt, int iters, unsigned long long* cyc) {
  cg::grid_group gg = cg::this_grid();
  long long c0 = clock64();
  for (int i = 0; i < iters; ++i) gg.sync();
  long long c1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) { cnt[0]++; cyc[0] = c1 - c0; }
}
__global__ void k_ctl(int* cnt, cudaGraphConditionalHandle h) { cudaGraphSetConditional(h, cnt[0] < 5); }
int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int* cnt; cudaMalloc(&cnt, 16); cudaMemset(cnt, 0, 16);
  unsigned long long* cyc; cudaMalloc(&cyc, 16);
  cudaStream_t st, cs; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
  cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(nsm); cfg.blockDim = dim3(256); cfg.stream = st;
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeCooperative; at[0].val.cooperative = 1; cfg.attrs = at; cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_coop, cnt, 1000, cyc); cudaStreamSynchronize(st);
  unsigned long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("direct coop launch: %s; grid.sync %.0f cycles\n", cudaGetErrorString(e), h / 1000.0);
  cudaGraph_t G; cudaGraphCreate(&G, 0);
  cudaGraphConditionalHandle hc; cudaGraphConditionalHandleCreate(&hc, G, 1, cudaGraphCondAssignDefault);
  cudaGraphNodeParams cp = {}; cp.type = cudaGraphNodeTypeConditional; cp.conditional.handle = hc; cp.conditional.type = cudaGraphCondTypeWhile; cp.conditional.size = 1;
  cudaGraphNode_t node; e = cudaGraphAddNode(&node, G, nullptr, 0, &cp); printf("while node: %s\n", cudaGetErrorString(e));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  e = cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal); printf("begin: %s\n", cudaGetErrorString(e));
  cfg.stream = cs;
  e = cudaLaunchKernelEx(&cfg, k_coop, cnt, 10, cyc); printf("capture coop: %s\n", cudaGetErrorString(e));
  k_ctl<<<1, 1, 0, cs>>>(cnt, hc);
  cudaGraph_t tmp; e = cudaStreamEndCapture(cs, &tmp); printf("end: %s\n", cudaGetErrorString(e));
  cudaGraphExec_t ex; e = cudaGraphInstantiate(&ex, G, 0); printf("instantiate: %s\n", cudaGetErrorString(e));
  cudaMemset(cnt, 0, 16);
  e = cudaGraphLaunch(ex, st); cudaStreamSynchronize(st); printf("launch: %s / %s\n", cudaGetErrorString(e), cudaGetErrorString(cudaGetLastError()));
  int hc2; cudaMemcpy(&hc2, cnt, 4, cudaMemcpyDeviceToHost); printf("iterations %d (expect 5)\n", hc2);
  return 0;
}
