// Probe: tcgen05.mma kind::f16 throughput for small N (decode shapes): M=128, K=16,
// A from TMEM, B from shared memory (SW128), one issuing thread, D rotating over TMEM.
#include <cstdio>
#include <cstdint>
#include "../paper_2511_10645_b200/csrc/umma.cuh"
using namespace paro;
PARO_DEV void mma_f16_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
template <int N, int SS>
__global__ void kmma(unsigned long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tbase_sh;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 32768; i += blockDim.x) smem[i] = 0;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&tbase_sh, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tbase_sh;
  unsigned long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = idesc_f16_f32(128, N);
    const uint64_t bdesc = smem_desc_sw128(smem);
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (SS)
          mma_f16_ss(tb + j * 32, smem_desc_sw128(smem + 8192) + (uint64_t)((j & 3) * 2), bdesc + (uint64_t)((j & 3) * 2), idesc, 1u);
        else
          mma_f16_ts(tb + (j & 3) * 16, tb + 256 + j * 8, bdesc + (uint64_t)((j & 3) * 2), idesc, 1u);
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    t1 = clock64();
    out[blockIdx.x] = (t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tb, 512); }
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 8 * 1024);
  unsigned long long h[4];
  const int iters = 2000;
#define RUN(NN, SS_)                                                                                     \
  {                                                                                                 \
    cudaFuncSetAttribute(kmma<NN, SS_>, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);          \
    for (int w = 0; w < 2; ++w) kmma<NN, SS_><<<148, 128, 40 * 1024>>>(d, iters);                         \
    cudaDeviceSynchronize();                                                                        \
    cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);                                                    \
    printf("%s N=%3d: %.2f cycles per MMA (M=128,K=16) -> %.1f dense MAC/clk/SM  (%s)\n", SS_ ? "A:smem" : "A:tmem", NN, h[0] / (iters * 8.0), \
           128.0 * NN * 16 / (h[0] / (iters * 8.0)), cudaGetErrorString(cudaGetLastError()));       \
  }
  RUN(8, 0) RUN(16, 0) RUN(64, 0) RUN(128, 0) RUN(8, 1) RUN(16, 1) RUN(64, 1) RUN(128, 1)
}
