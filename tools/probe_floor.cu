// Floor probe: what a lean one-wave streaming kernel costs per launch on this B200, in a CUDA
// graph with programmatic dependent launch (PDL).  Each CTA bulk-copies (TMA engine) its
// contiguous share of a weight-sized buffer through a shared-memory ring and touches every
// 16 B; buffers cycle through a pool larger than L2.  Prints us per launch and GB/s.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -I paper_2511_10645_b200/csrc -o /tmp/pf tools/probe_floor.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include "ptx.cuh"
using namespace paro;

#ifndef HALF
#define HALF 0  // 1: half-SM footprint (8 consumer warps, 3 x 32 KB ring) so the next PDL launch co-resides
#endif
#ifndef CLUSTER
#define CLUSTER 1
#endif
constexpr int NW = HALF ? 8 : 16;
constexpr uint32_t STG = 32 * 1024;
constexpr int S = HALF ? 3 : 6;

__global__ void __launch_bounds__((NW + 1) * 32, HALF ? 2 : 1) stream_k(const uint8_t* base, uint32_t per_cta, const uint4* x, float* out, int pdl, int prefetch_before_wait) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * STG);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], NW); }
    fence_mbar_init();
  }
  __syncthreads();
  if (pdl) pdl_launch_dependents();
  const uint8_t* src = base + static_cast<size_t>(blockIdx.x) * per_cta;
  const int nch = (per_cta + STG - 1) / STG;
  if (warp == NW) {
    if (pdl && !prefetch_before_wait) pdl_wait();
    if (lane == 0) {
      const uint64_t pol = l2_evict_first_policy();
      for (int i = 0; i < nch; ++i) {
        const int slot = i % S;
        if (i >= S) mbar_wait(&empty[slot], ((i / S) & 1) ^ 1);
        const uint32_t nb = min(STG, per_cta - i * STG);
        mbar_arrive_expect_tx(&full[slot], nb);
        bulk_g2s(smem + slot * STG, src + static_cast<size_t>(i) * STG, nb, &full[slot], pol);
      }
    }
    return;
  }
  if (pdl) pdl_wait();
  uint4 acc = x[threadIdx.x & 255];
  for (int i = 0; i < nch; ++i) {
    const int slot = i % S;
    mbar_wait(&full[slot], (i / S) & 1);
    const uint32_t nb = min(STG, per_cta - i * STG);
    const uint4* p = reinterpret_cast<const uint4*>(smem + slot * STG);
    for (uint32_t k = threadIdx.x; k < nb / 16; k += NW * 32) {
      uint4 v = p[k];
      acc.x ^= v.x; acc.y += v.y; acc.z ^= v.z; acc.w += v.w;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345u) out[blockIdx.x * 1024 + threadIdx.x] = 1.f;
  if (threadIdx.x == 0) out[blockIdx.x] = acc.x;
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = S * STG + 2 * S * 8;
  cudaFuncSetAttribute(stream_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const size_t sizes[] = {0, 8716288, 30507008, 61014016};
  uint4* x; float* out; cudaMalloc(&x, 4096); cudaMalloc(&out, sms * 1024 * 4 * 2);
  const size_t pool_bytes = 640ull << 20;
  uint8_t* pool; cudaMalloc(&pool, pool_bytes); cudaMemset(pool, 1, pool_bytes);
  cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  printf("HALF=%d CLUSTER=%d\n", HALF, CLUSTER);
  for (int pdl = 1; pdl < 2; ++pdl)
    for (int pf = 1; pf < 2; ++pf)
      for (size_t bytes : sizes) {
        uint32_t per = (uint32_t)(((bytes + sms - 1) / sms + 15) / 16 * 16);
        if (per == 0) per = 16;
        const size_t span = (size_t)per * sms;
        const int nbuf = (int)std::max<size_t>(1, pool_bytes / std::max<size_t>(span, 1));
        const int reps = 40;
        cudaGraph_t g; cudaGraphExec_t ge;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
        for (int r = 0; r < reps; ++r) {
          cudaLaunchConfig_t cfg{};
          cfg.gridDim = dim3(sms); cfg.blockDim = dim3((NW + 1) * 32); cfg.dynamicSmemBytes = smem; cfg.stream = st;
          cudaLaunchAttribute at[2]; int na = 0;
          if (pdl) { at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[na].val.programmaticStreamSerializationAllowed = 1; ++na; }
          if (CLUSTER > 1) { at[na].id = cudaLaunchAttributeClusterDimension; at[na].val.clusterDim.x = CLUSTER;
            at[na].val.clusterDim.y = 1; at[na].val.clusterDim.z = 1; ++na; }
          cfg.attrs = at; cfg.numAttrs = na;
          const uint8_t* b = pool + (size_t)(r % std::min(nbuf, 64)) * span;
          cudaLaunchKernelEx(&cfg, stream_k, b, per, (const uint4*)x, out, pdl, pf);
        }
        cudaStreamEndCapture(st, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaGraphLaunch(ge, st); cudaStreamSynchronize(st);
        float best = 1e30f;
        for (int it = 0; it < 5; ++it) {
          cudaEventRecord(e0, st); cudaGraphLaunch(ge, st); cudaEventRecord(e1, st); cudaEventSynchronize(e1);
          float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms);
        }
        const double us = best * 1e3 / reps;
        printf("pdl=%d prefetch_before_wait=%d bytes=%10zu nbuf=%3d: %7.3f us/launch  %7.1f GB/s\n", pdl, pf, bytes,
               std::min(nbuf, 64), us, bytes / us / 1e3);
        cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
      }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
