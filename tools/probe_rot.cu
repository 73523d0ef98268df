// Probe: latency of an 8-layer Givens rotation chain on one 128-float group:
//  mode 0: shared memory, 4 LDS + 8 FMA + 4 STS + __syncwarp per layer
//  mode 1: same without __syncwarp (timing only)
//  mode 2: registers + 4 shfl.idx + runtime 4-way selects per layer (timing only)
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ float sel4(float a, float b, float c, float d, uint32_t k) {
  const float lo = (k & 1) ? b : a, hi = (k & 1) ? d : c;
  return (k & 2) ? hi : lo;
}
template <int MODE>
__global__ void krot(const uint32_t* __restrict__ idx, float* out, unsigned long long* cyc, int reps, int active_warps,
                     int B = 1, const float4* __restrict__ csg = nullptr) {
  extern __shared__ float sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp >= active_warps) return;
  float* scr = sm + warp * 132;
  for (int i = lane; i < 128; i += 32) scr[i] = i * 0.01f;
  uint32_t ix[8];
  for (int t = 0; t < 8; ++t) ix[t] = idx[t * 32 + lane];
  float v0 = lane, v1 = lane + 1, v2 = lane + 2, v3 = lane + 3;
  float4 csr[8];
  for (int t = 0; t < 8; ++t) csr[t] = csg ? csg[t * 32 + lane] : make_float4(0.8f, 0.6f, 0.8f, 0.6f);
  __syncwarp();
  unsigned long long c0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const uint32_t i0 = ix[t] & 0xff, j0 = (ix[t] >> 8) & 0xff, i1 = (ix[t] >> 16) & 0xff, j1 = ix[t] >> 24;
      const float c = 0.8f, s = 0.6f;
      if (MODE == 3) {  // the decode kernel's form: runtime token loop, (cos, sin) from registers
        for (int b = 0; b < B; ++b) {
          float* sb = scr + b * 132;
          const float a0 = sb[i0], b0 = sb[j0];
          const float a1 = sb[i1], b1 = sb[j1];
          sb[i0] = csr[t].x * a0 - csr[t].y * b0;
          sb[j0] = csr[t].y * a0 + csr[t].x * b0;
          sb[i1] = csr[t].z * a1 - csr[t].w * b1;
          sb[j1] = csr[t].w * a1 + csr[t].z * b1;
        }
        __syncwarp();
      } else if (MODE < 2) {
        const float a0 = scr[i0], b0 = scr[j0], a1 = scr[i1], b1 = scr[j1];
        scr[i0] = c * a0 - s * b0;
        scr[j0] = s * a0 + c * b0;
        scr[i1] = c * a1 - s * b1;
        scr[j1] = s * a1 + c * b1;
        if (MODE == 0) __syncwarp();
      } else {
        const float r0 = __shfl_sync(0xffffffffu, v0, i0 & 31);
        const float r1 = __shfl_sync(0xffffffffu, v1, j0 & 31);
        const float r2 = __shfl_sync(0xffffffffu, v2, i1 & 31);
        const float r3 = __shfl_sync(0xffffffffu, v3, j1 & 31);
        const float a0 = sel4(r0, r1, r2, r3, i0 >> 5), b0 = sel4(r0, r1, r2, r3, j0 >> 5);
        const float a1 = sel4(r0, r1, r2, r3, i1 >> 5), b1 = sel4(r0, r1, r2, r3, j1 >> 5);
        v0 = c * a0 - s * b0;
        v1 = s * a0 + c * b0;
        v2 = c * a1 - s * b1;
        v3 = s * a1 + c * b1;
      }
    }
  }
  unsigned long long c1 = clock64();
  if (lane == 0) cyc[blockIdx.x * 32 + warp] = (c1 - c0) / reps;
  out[blockIdx.x * blockDim.x + threadIdx.x] = scr[lane] + v0 + v1 + v2 + v3;
}
int main() {
  uint32_t h[8 * 32];
  for (int t = 0; t < 8; ++t) {
    const int m = 1 << (t % 6 + 1);
    for (int l = 0; l < 32; ++l) {
      int a = 0, cnt = 0;
      for (int c = 0; c < 64; ++c)
        if (!(c & m)) { if (cnt == l) { a = c; break; } ++cnt; }
      h[t * 32 + l] = a | ((a ^ m) << 8) | ((a + 64) << 16) | (((a + 64) ^ m) << 24);
    }
  }
  uint32_t* d; float* o; unsigned long long* cyc;
  cudaMalloc(&d, sizeof(h)); cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaMalloc(&o, 1 << 22); cudaMalloc(&cyc, 8 * 4096);
  unsigned long long hc[64];
  float4* csd; cudaMalloc(&csd, 8 * 32 * 16);
  float4 hcs[256]; for (int i = 0; i < 256; ++i) hcs[i] = make_float4(0.8f, 0.6f, 0.8f, 0.6f);
  cudaMemcpy(csd, hcs, sizeof(hcs), cudaMemcpyHostToDevice);
  for (int aw = 1; aw <= 8; aw *= 2) {
    for (int w = 0; w < 2; ++w) krot<3><<<148, 288, 8 * 1024>>>(d, o, cyc, 100, aw, 1, csd);
    cudaDeviceSynchronize();
    cudaMemcpy(hc, cyc, 8 * 9, cudaMemcpyDeviceToHost);
    printf("mode 3 (kernel form, B=1) active warps/CTA %d: cycles per layer %.1f  err=%s\n", aw, hc[0] / 8.0,
           cudaGetErrorString(cudaGetLastError()));
  }
  for (int mode = 0; mode < 3; ++mode)
    for (int aw = 1; aw <= 8; aw *= 2) {
      for (int w = 0; w < 2; ++w) {
        if (mode == 0) krot<0><<<148, 288, 8 * 1024>>>(d, o, cyc, 100, aw);
        if (mode == 1) krot<1><<<148, 288, 8 * 1024>>>(d, o, cyc, 100, aw);
        if (mode == 2) krot<2><<<148, 288, 8 * 1024>>>(d, o, cyc, 100, aw);
      }
      cudaDeviceSynchronize();
      cudaMemcpy(hc, cyc, 8 * 9, cudaMemcpyDeviceToHost);
      printf("mode %d active warps/CTA %d: cycles per layer %.1f  err=%s\n", mode, aw, hc[0] / 8.0,
             cudaGetErrorString(cudaGetLastError()));
    }
}
