// Probe: do legacy HMMA (mma.sync) and FFMA / LOP3 from other warps of the same SM
// sub-partition overlap?  Warps [0, nh) run HMMA chains, warps [nh, nw) run FFMA or LOP3
// chains; report each group's rate alone and together.
#include <cstdio>
#include <cstdint>
#include "../paper_2511_10645_b200/csrc/ptx.cuh"
using namespace paro;
template <int OTHER>  // 0: FFMA, 1: LOP3
__global__ void kmix(float* out, unsigned long long* cyc, int iters, int nh, int run_h, int run_o) {
  const int warp = threadIdx.x >> 5;
  unsigned long long c0 = clock64();
  float r = 0.f;
  if (warp < nh) {
    if (run_h) {
      uint32_t a = 0x00030005u + threadIdx.x, b = 0x3c003c00u;
      float D[8][4] = {};
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; j++) mma_16816(D[j], a + j, a ^ j, a, a + it, b, b);
      }
      for (int j = 0; j < 8; j++) r += D[j][0];
    }
  } else if (run_o) {
    float f[8];
    uint32_t u[8];
    for (int j = 0; j < 8; ++j) { f[j] = threadIdx.x * 0.1f + j; u[j] = threadIdx.x * 7u + j; }
    for (int it = 0; it < iters * 10; ++it) {
#pragma unroll
      for (int j = 0; j < 8; j++) {
        if (OTHER == 0) f[j] = fmaf(f[j], 0.999f, 0.5f);
        else u[j] = (u[j] & 0x0F0F0F0Fu) ^ (u[j] >> 3);
      }
    }
    for (int j = 0; j < 8; ++j) r += f[j] + u[j];
  }
  unsigned long long c1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 32 + warp] = c1 - c0;
}
int main() {
  float* o; unsigned long long* cyc; cudaMalloc(&o, 1 << 22); cudaMalloc(&cyc, 8 * 148 * 32);
  const int iters = 2000, nw = 16, nh = 8;
  unsigned long long h[32];
  for (int other = 0; other < 2; ++other)
    for (int mode = 0; mode < 3; ++mode) {  // 0: HMMA alone, 1: other alone, 2: both
      const int rh = mode != 1, ro = mode != 0;
      for (int rep = 0; rep < 2; ++rep) {
        if (other == 0) kmix<0><<<148, nw * 32>>>(o, cyc, iters, nh, rh, ro);
        else kmix<1><<<148, nw * 32>>>(o, cyc, iters, nh, rh, ro);
        cudaDeviceSynchronize();
      }
      cudaMemcpy(h, cyc, 8 * 32, cudaMemcpyDeviceToHost);
      unsigned long long th = 0, to = 0;
      for (int w = 0; w < nh; ++w) th = h[w] > th ? h[w] : th;
      for (int w = nh; w < nw; ++w) to = h[w] > to ? h[w] : to;
      printf("%s %-10s: HMMA warps %llu cycles (%.2f HMMA/clk/SMSP), other warps %llu cycles (%.2f instr/clk/SMSP)\n",
             other ? "LOP3" : "FFMA", mode == 0 ? "HMMA only" : mode == 1 ? "other only" : "both", th,
             rh ? (double)iters * 8 * nh / 4 / th : 0.0, to, ro ? (double)iters * 10 * 8 * (nw - nh) / 4 / to : 0.0);
    }
}
