// Probe: cost per dependent tiny kernel — stream launches vs graph chain vs conditional WHILE.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void tick(int* c) { if (threadIdx.x == 0 && blockIdx.x == 0) c[0]++; }
__global__ void tickw(int* c, cudaGraphConditionalHandle h, int lim) {
  if (threadIdx.x == 0 && blockIdx.x == 0) { c[0]++; cudaGraphSetConditional(h, c[0] < lim); }
}
int main() {
  int* c; cudaMalloc(&c, 16);
  cudaStream_t s; cudaStreamCreate(&s);
  cudaEvent_t t0, t1; cudaEventCreate(&t0); cudaEventCreate(&t1);
  const int K = 200;
  float ms;
  for (int grid : {1, 148}) {
    // (a) stream launches
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(t0, s);
      for (int i = 0; i < K; ++i) tick<<<grid, 128, 0, s>>>(c);
      cudaEventRecord(t1, s); cudaEventSynchronize(t1); cudaEventElapsedTime(&ms, t0, t1);
    }
    printf("grid %3d stream launches: %.2f us/kernel\n", grid, ms * 1e3 / K);
    // (b) graph chain
    cudaGraph_t g; cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < K; ++i) tick<<<grid, 128, 0, s>>>(c);
    cudaStreamEndCapture(s, &g);
    cudaGraphExec_t ex; cudaGraphInstantiate(&ex, g, 0);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(t0, s); cudaGraphLaunch(ex, s); cudaEventRecord(t1, s); cudaEventSynchronize(t1);
      cudaEventElapsedTime(&ms, t0, t1);
    }
    printf("grid %3d graph chain:      %.2f us/kernel\n", grid, ms * 1e3 / K);
    // (c) WHILE with a 4-kernel body
    cudaGraph_t gw; cudaGraphCreate(&gw, 0);
    cudaGraphConditionalHandle h; cudaGraphConditionalHandleCreate(&h, gw, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams cp = {cudaGraphNodeTypeConditional};
    cp.conditional.handle = h; cp.conditional.type = cudaGraphCondTypeWhile; cp.conditional.size = 1;
    cudaGraphNode_t wn; cudaGraphAddNode(&wn, gw, nullptr, 0, &cp);
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    cudaGraphNode_t prev = nullptr;
    int lim = K / 4;
    for (int i = 0; i < 4; ++i) {
      cudaKernelNodeParams kp = {};
      void* a1[] = {&c}; void* a2[] = {&c, &h, &lim};
      kp.func = (i < 3) ? (void*)tick : (void*)tickw; kp.gridDim = grid; kp.blockDim = 128; kp.kernelParams = (i < 3) ? a1 : a2;
      cudaGraphNode_t n; cudaGraphAddKernelNode(&n, body, prev ? &prev : nullptr, prev ? 1 : 0, &kp); prev = n;
    }
    cudaGraphExec_t exw; cudaError_t e = cudaGraphInstantiate(&exw, gw, 0);
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(c, 0, 16);
      cudaEventRecord(t0, s); cudaGraphLaunch(exw, s); cudaEventRecord(t1, s); cudaEventSynchronize(t1);
      cudaEventElapsedTime(&ms, t0, t1);
    }
    printf("grid %3d WHILE(4-kernel body) x%d: %.2f us/kernel  (%s)\n", grid, lim, ms * 1e3 / (4 * lim), cudaGetErrorString(e));
  }
  return 0;
}
