// Probe: per-kernel cost of a dependent chain inside a conditional WHILE body captured from a stream,
// with and without programmatic dependent launch (PDL: launch attribute + griddepcontrol).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }
template <bool TRIG>
__global__ void tick(int* c, int spin) {
  pdl_wait();
  if (TRIG) pdl_trigger();
  long long t0 = clock64();
  while (clock64() - t0 < spin) {}
  if (threadIdx.x == 0 && blockIdx.x == 0) c[1]++;
}
template <bool TRIG>
__global__ void tickw(int* c, cudaGraphConditionalHandle h, int lim) {
  pdl_wait();
  if (threadIdx.x == 0 && blockIdx.x == 0) { c[0]++; cudaGraphSetConditional(h, c[0] < lim); }
}
template <bool TRIG>
void launch(cudaStream_t s, int grid, int pdl, int* c, int spin) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid; cfg.blockDim = 128; cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at; cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, tick<TRIG>, c, spin);
}
int main() {
  int* c; cudaMalloc(&c, 16);
  cudaStream_t s, cs; cudaStreamCreate(&s); cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
  cudaEvent_t t0, t1; cudaEventCreate(&t0); cudaEventCreate(&t1);
  const int lim = 100;
  for (int spin : {0, 4000}) for (int grid : {1, 148, 296}) for (int mode = 0; mode < 3; ++mode) {
    const int pdl = mode > 0; const bool trig = mode == 2;
    cudaGraph_t gw; cudaGraphCreate(&gw, 0);
    cudaGraphConditionalHandle h; cudaGraphConditionalHandleCreate(&h, gw, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams cp = {cudaGraphNodeTypeConditional};
    cp.conditional.handle = h; cp.conditional.type = cudaGraphCondTypeWhile; cp.conditional.size = 1;
    cudaGraphNode_t wn; cudaGraphAddNode(&wn, gw, nullptr, 0, &cp);
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    cudaError_t e1 = cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < 7; ++i) { if (trig) launch<true>(cs, grid, pdl, c, spin); else launch<false>(cs, grid, pdl, c, spin); }
    {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = 1; cfg.blockDim = 32; cfg.stream = cs;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at; cfg.numAttrs = pdl ? 1 : 0;
      cudaLaunchKernelEx(&cfg, tickw<false>, c, h, lim);
    }
    cudaGraph_t tmp; cudaError_t e2 = cudaStreamEndCapture(cs, &tmp);
    cudaGraphExec_t exw; cudaError_t e = cudaGraphInstantiate(&exw, gw, 0);
    float ms = 0;
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(c, 0, 16);
      cudaEventRecord(t0, s); cudaGraphLaunch(exw, s); cudaEventRecord(t1, s); cudaEventSynchronize(t1);
      cudaEventElapsedTime(&ms, t0, t1);
    }
    int hc[2]; cudaMemcpy(hc, c, 8, cudaMemcpyDeviceToHost);
    printf("spin %5d grid %3d %-12s: %.2f us/kernel  (iters %d, ticks %d; %s %s %s %s)\n", spin, grid,
           mode == 0 ? "plain" : (mode == 1 ? "pdl" : "pdl+trigger"), ms * 1e3 / (8 * lim), hc[0], hc[1],
           cudaGetErrorString(e1), cudaGetErrorString(e2), cudaGetErrorString(e), cudaGetErrorString(cudaGetLastError()));
    cudaGraphExecDestroy(exw); cudaGraphDestroy(gw);
  }
  return 0;
}
