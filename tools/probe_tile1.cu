// Tile-loop probe for the K-split decode kernel's IMMA tile body (gemv1.cu, B = 1): each warp
// runs `iters` tiles on shared-memory-resident data; prints cycles per tile per warp and tiles per
// microsecond per SM for 1..16 warps per CTA (one CTA per SM).
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>

__device__ __forceinline__ void mma_u8s8(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
  asm("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int MODE>
__global__ void k(int iters, float* out, long long* cyc) {
  __shared__ __align__(16) uint8_t tiles[8][2048 + 128];
  __shared__ __align__(16) uint8_t xp[8 * 256];
  __shared__ float pw[16][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gq = lane >> 2, tq = lane & 3;
  for (int i = threadIdx.x; i < 8 * (2048 + 128) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(tiles)[i] = i * 2654435761u;
  for (int i = threadIdx.x; i < 8 * 256 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(xp)[i] = i * 40503u;
  for (int i = threadIdx.x; i < 16 * 256; i += blockDim.x) (&pw[0][0])[i] = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int ti = (it + warp) & 7;
    const uint8_t* sb = tiles[ti];
    const uint8_t* tc = sb + gq * 64 + tq * 16;
    uint4 w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) w[q] = *reinterpret_cast<const uint4*>(tc + q * 512);
    uint4 bA = make_uint4(0u, 0u, 0u, 0u), bB = bA;
    if (gq < 2) {
      const uint8_t* bp = xp + ti * 256 + tq * 64 + gq * 32;
      bA = *reinterpret_cast<const uint4*>(bp);
      bB = *reinterpret_cast<const uint4*>(bp + 16);
    }
    constexpr uint32_t ML = 0x0f0f0f0fu, MH = 0xf0f0f0f0u;
    int Dl[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}}, Dh[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const uint4 r0 = w[2 * hh], r1 = w[2 * hh + 1];
      mma_u8s8(Dl[hh], r0.x & ML, r1.x & ML, r0.y & ML, r1.y & ML, bA.x, bA.y);
      mma_u8s8(Dl[hh], r0.z & ML, r1.z & ML, r0.w & ML, r1.w & ML, bA.z, bA.w);
      mma_u8s8(Dh[hh], r0.x & MH, r1.x & MH, r0.y & MH, r1.y & MH, bB.x, bB.y);
      mma_u8s8(Dh[hh], r0.z & MH, r1.z & MH, r0.w & MH, r1.w & MH, bB.z, bB.w);
    }
    if (MODE == 1 || tq == 0) {
      const uint2 sp = *reinterpret_cast<const uint2*>(sb + 2048 + gq * 8);
      const uint32_t zw = *reinterpret_cast<const uint16_t*>(sb + 2048 + 64 + gq * 2);
      const float2 Sa = __half22float2(*reinterpret_cast<const __half2*>(&sp.x));
      const float2 Sb = __half22float2(*reinterpret_cast<const __half2*>(&sp.y));
      const float Sr[4] = {Sa.x, Sa.y, Sb.x, Sb.y};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int hh = q >> 1, e = (q & 1) * 2;
        const int zq = static_cast<int>((zw >> (4 * q)) & 15u);
        const int I = Dl[hh][e] * 256 + Dl[hh][e + 1] + ((Dh[hh][e] * 256 + Dh[hh][e + 1]) >> 4) - zq * 7;
        pw[warp][(ti * 32 + gq + 8 * q) & 255] += Sr[q] * 1.5f * static_cast<float>(I);
      }
    }
  }
  long long t1 = clock64();
  if (lane == 0) cyc[blockIdx.x * 32 + warp] = t1 - t0;
  if (threadIdx.x == 0) out[blockIdx.x] = pw[0][0] + pw[warp][5];
}

int main() {
  float* out; long long* cyc; cudaMalloc(&out, 4096 * 4); cudaMalloc(&cyc, 148 * 32 * 8);
  long long h[148 * 32];
  const int iters = 2000;
  for (int nw : {1, 2, 4, 8, 16}) {
    k<0><<<148, nw * 32>>>(iters, out, cyc);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    k<0><<<148, nw * 32>>>(iters, out, cyc);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("warps/SM %2d: %.0f cycles per tile per warp, %.1f tiles/us/SM (%.0f weights/clk/SM at 1.965 GHz)\n", nw,
           (double)h[0] / iters, nw * iters / (ms * 1e3), nw * iters * 4096.0 / (ms * 1e-3) / 1.965e9);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
