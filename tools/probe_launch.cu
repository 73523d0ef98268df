// Probe: per-launch cost of back-to-back kernels in a CUDA graph for the launch shapes the
// decode kernel uses (grid, block, dynamic smem, cluster), empty body vs a 2 us body.
#include <cstdio>
#include <cstdint>
__global__ void kempty(int* p) {
  extern __shared__ int sm[];
  if (threadIdx.x == 0 && blockIdx.x == 0 && p[0] == 12345) p[1] = sm[0];
}
int main() {
  int* d; cudaMalloc(&d, 64); cudaMemset(d, 0, 64);
  cudaFuncSetAttribute(kempty, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  struct Cfg { int grid, block, smem, cl; } cfgs[] = {
      {148, 288, 0, 1}, {296, 288, 0, 1}, {264, 288, 106 * 1024, 8}, {296, 288, 106 * 1024, 2},
      {144, 544, 210 * 1024, 8}, {148, 544, 210 * 1024, 4}, {148, 544, 210 * 1024, 1}, {264, 288, 106 * 1024, 1}};
  cudaStream_t s; cudaStreamCreate(&s);
  for (auto c : cfgs) {
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(c.grid); lc.blockDim = dim3(c.block); lc.dynamicSmemBytes = c.smem; lc.stream = s;
    cudaLaunchAttribute at; at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = c.cl; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
    if (c.cl > 1) { lc.attrs = &at; lc.numAttrs = 1; }
    cudaGraph_t g; cudaGraphExec_t ge;
    const int n = 200;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < n; ++i) cudaLaunchKernelEx(&lc, kempty, d);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, s); cudaGraphLaunch(ge, s); cudaEventRecord(e1, s); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("grid %d block %d smem %dKB cluster %d: %.2f us per empty launch  (%s)\n", c.grid, c.block, c.smem / 1024, c.cl,
           ms * 1000 / n, cudaGetErrorString(cudaGetLastError()));
  }
}
