// Probe: conditional WHILE graph nodes with a nested WHILE, set from device code.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void body_inner(int* cnt, cudaGraphConditionalHandle h) {
  cnt[1]++;
  cudaGraphSetConditional(h, (cnt[1] % 3) != 0);
}
__global__ void body_outer(int* cnt, cudaGraphConditionalHandle h) {
  cnt[0]++;
  cudaGraphSetConditional(h, cnt[0] < 5);
}
__global__ void init_inner(int* cnt, cudaGraphConditionalHandle h) { cudaGraphSetConditional(h, 1); }
int main() {
  int* cnt; cudaMalloc(&cnt, 16); cudaMemset(cnt, 0, 16);
  cudaGraph_t g; cudaGraphCreate(&g, 0);
  cudaGraphConditionalHandle ho, hi;
  cudaGraphConditionalHandleCreate(&ho, g, 1, cudaGraphCondAssignDefault);
  cudaGraphNodeParams cp = {cudaGraphNodeTypeConditional};
  cp.conditional.handle = ho; cp.conditional.type = cudaGraphCondTypeWhile; cp.conditional.size = 1;
  cudaGraphNode_t wo;
  cudaError_t e = cudaGraphAddNode(&wo, g, nullptr, 0, &cp);
  printf("add outer while: %s\n", cudaGetErrorString(e));
  cudaGraph_t bo = cp.conditional.phGraph_out[0];
  // outer body: init_inner -> inner WHILE -> body_outer
  cudaGraphConditionalHandleCreate(&hi, bo, 0, 0);
  cudaKernelNodeParams kp = {}; void* a1[] = {&cnt, &hi};
  kp.func = (void*)init_inner; kp.gridDim = 1; kp.blockDim = 1; kp.kernelParams = a1;
  cudaGraphNode_t n1; e = cudaGraphAddKernelNode(&n1, bo, nullptr, 0, &kp); printf("init_inner: %s\n", cudaGetErrorString(e));
  cudaGraphNodeParams ci = {cudaGraphNodeTypeConditional};
  ci.conditional.handle = hi; ci.conditional.type = cudaGraphCondTypeWhile; ci.conditional.size = 1;
  cudaGraphNode_t wi; e = cudaGraphAddNode(&wi, bo, &n1, 1, &ci); printf("nested while: %s\n", cudaGetErrorString(e));
  cudaGraph_t bi = ci.conditional.phGraph_out[0];
  cudaKernelNodeParams kb = {}; void* a2[] = {&cnt, &hi};
  kb.func = (void*)body_inner; kb.gridDim = 1; kb.blockDim = 1; kb.kernelParams = a2;
  cudaGraphNode_t n2; e = cudaGraphAddKernelNode(&n2, bi, nullptr, 0, &kb); printf("inner body: %s\n", cudaGetErrorString(e));
  cudaKernelNodeParams ko = {}; void* a3[] = {&cnt, &ho};
  ko.func = (void*)body_outer; ko.gridDim = 1; ko.blockDim = 1; ko.kernelParams = a3;
  cudaGraphNode_t n3; e = cudaGraphAddKernelNode(&n3, bo, &wi, 1, &ko); printf("outer body: %s\n", cudaGetErrorString(e));
  cudaGraphExec_t ex; e = cudaGraphInstantiate(&ex, g, 0); printf("instantiate: %s\n", cudaGetErrorString(e));
  cudaEvent_t t0, t1; cudaEventCreate(&t0); cudaEventCreate(&t1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(cnt, 0, 16);
    cudaEventRecord(t0);
    e = cudaGraphLaunch(ex, 0); cudaEventRecord(t1); cudaEventSynchronize(t1);
    int h[2]; cudaMemcpy(h, cnt, 8, cudaMemcpyDeviceToHost);
    float ms; cudaEventElapsedTime(&ms, t0, t1);
    printf("launch: %s  outer=%d inner=%d  (expect 5, 15)  %.1f us\n", cudaGetErrorString(e), h[0], h[1], ms * 1e3);
  }
  return 0;
}
