// Probe: throughput of the decode kernel's per-tile inner loop (32 rows x 128 k, B=1) with
// the data resident in shared memory, 15 warps / CTA, 1 CTA / SM.  Variants:
//   0: full tile (4 LDS.128 codes, 4 LDS.128 B fragments, 16 HMMA, epilogue)
//   1: no epilogue (accumulate D only)
//   2: FHFMA (fp32 += f16 * f16) instead of HMMA, epilogue per lane-row, quad reduction deferred
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include "../paper_2511_10645_b200/csrc/ptx.cuh"
using namespace paro;
__device__ __forceinline__ float fl(uint32_t a, uint32_t b, float c) {
  float d;
  asm("{.reg .f16 a0,a1,b0,b1;\n mov.b32 {a0,a1},%1;\n mov.b32 {b0,b1},%2;\n fma.rn.f32.f16 %0,a0,b0,%3;}" : "=f"(d) : "r"(a), "r"(b), "f"(c));
  return d;
}
__device__ __forceinline__ float fh(uint32_t a, uint32_t b, float c) {
  float d;
  asm("{.reg .f16 a0,a1,b0,b1;\n mov.b32 {a0,a1},%1;\n mov.b32 {b0,b1},%2;\n fma.rn.f32.f16 %0,a1,b1,%3;}" : "=f"(d) : "r"(a), "r"(b), "f"(c));
  return d;
}
template <int V>
__global__ void __launch_bounds__(480, 1) ktile(float* out, unsigned long long* cyc, int ntiles) {
  extern __shared__ __align__(16) uint8_t sm[];
  // 32 tiles of codes (64 KB) + 32 groups of B fragments (32 x 256 B) + scales/zeros/xsum
  uint8_t* codes = sm;
  uint8_t* frag = sm + 65536;
  uint8_t* sc = frag + 8192;
  uint8_t* zz = sc + 2048;
  float* xsum = reinterpret_cast<float*>(zz + 512);
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(codes)[i] = 0x5a3c1e7bu * (i + 1);
  for (int i = threadIdx.x; i < (8192 + 2048 + 512 + 1024) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(frag)[i] = 0x3c003c00u;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, NW = blockDim.x >> 5;
  const int gq = lane >> 2, t = lane & 3;
  const uint32_t cbase = smem_u32(codes), fbase = smem_u32(frag), sbase = smem_u32(sc), zbase = smem_u32(zz),
                 xbase = smem_u32(xsum);
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  float Dk[2][4] = {};
  unsigned long long c0 = clock64();
  for (int it = warp; it < ntiles; it += NW) {
    const int i = it & 31, g = it & 31;
    const uint32_t ca = cbase + i * 2048 + lane * 16;
    uint4 w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) w[q] = lds128_a(ca + q * 512);
    uint32_t bf[16];
    const uint32_t xa = fbase + g * 256 + t * 16;
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) {
      const uint4 v = lds128_a(xa + ii * 64);
      bf[4 * ii] = v.x; bf[4 * ii + 1] = v.y; bf[4 * ii + 2] = v.z; bf[4 * ii + 3] = v.w;
    }
    if (V < 2 || V == 3) {
      float D1[2][4], D16[2][4];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t w0[4] = {w[2 * h].x, w[2 * h].y, w[2 * h].z, w[2 * h].w};
        const uint32_t w1[4] = {w[2 * h + 1].x, w[2 * h + 1].y, w[2 * h + 1].z, w[2 * h + 1].w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t x = w0[j], y = w1[j];
          uint32_t x0, y0, x8, y8, x1, y1, x9, y9;
          x0 = x & 0x000F000Fu; y0 = y & 0x000F000Fu; x1 = x & 0x00F000F0u; y1 = y & 0x00F000F0u;
          if (V == 3) {  // upper nibbles: AND on the ALU pipe, >> 8 as IMAD.HI on the FMA pipe
            x8 = __umulhi(x & 0x0F000F00u, 1u << 24); y8 = __umulhi(y & 0x0F000F00u, 1u << 24);
            x9 = __umulhi(x & 0xF000F000u, 1u << 24); y9 = __umulhi(y & 0xF000F000u, 1u << 24);
          } else {
            x8 = (x >> 8) & 0x000F000Fu; y8 = (y >> 8) & 0x000F000Fu; x9 = (x >> 8) & 0x00F000F0u; y9 = (y >> 8) & 0x00F000F0u;
          }
          if (j == 0) {
            mma_16816_z(D1[h], x0, y0, x8, y8, bf[0], bf[1]);
            mma_16816_z(D16[h], x1, y1, x9, y9, bf[2], bf[3]);
          } else {
            mma_16816(D1[h], x0, y0, x8, y8, bf[4 * j], bf[4 * j + 1]);
            mma_16816(D16[h], x1, y1, x9, y9, bf[4 * j + 2], bf[4 * j + 3]);
          }
        }
      }
      if (V == 0 || V == 3) {
        const uint2 sp = lds_u64_a(sbase + i * 64 + gq * 8);
        const uint32_t zw = lds_u16z_a(zbase + i * 16 + gq * 2);
        const float2 Sa = __half22float2(*reinterpret_cast<const __half2*>(&sp.x));
        const float2 Sb = __half22float2(*reinterpret_cast<const __half2*>(&sp.y));
        const float2 X2 = lds_f2_a(xbase + (g * 8 + 2 * t) * 4);
        const float Sr[4] = {Sa.x, Sa.y, Sb.x, Sb.y};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float zq = static_cast<float>((zw >> (4 * q)) & 15u);
          const int h = q >> 1, e = (q & 1) * 2;
          acc[4 * h + e] = fmaf(Sr[q], fmaf(fmaf(D16[h][e], 0.0625f, D1[h][e]), 16777216.f, -zq * X2.x), acc[4 * h + e]);
          acc[4 * h + e + 1] = fmaf(Sr[q], fmaf(fmaf(D16[h][e + 1], 0.0625f, D1[h][e + 1]), 16777216.f, -zq * X2.y), acc[4 * h + e + 1]);
        }
      } else {
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int e = 0; e < 4; ++e) Dk[h][e] += D1[h][e] + D16[h][e];
      }
    } else {
      // FHFMA: lane's 4 rows (gq + 8q) x its 32 channels (quad t); x' pairs are bf[]
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float tl = 0.f, th = 0.f;
        const uint32_t wq[4] = {w[q].x, w[q].y, w[q].z, w[q].w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t x = wq[j], x8 = x >> 8;
          tl = fl(x & 0x000F000Fu, bf[4 * j], tl);
          th = fl(x & 0x00F000F0u, bf[4 * j + 2], th);
          tl = fh(x & 0x000F000Fu, bf[4 * j], tl);
          th = fh(x & 0x00F000F0u, bf[4 * j + 2], th);
          tl = fl(x8 & 0x000F000Fu, bf[4 * j + 1], tl);
          th = fl(x8 & 0x00F000F0u, bf[4 * j + 3], th);
          tl = fh(x8 & 0x000F000Fu, bf[4 * j + 1], tl);
          th = fh(x8 & 0x00F000F0u, bf[4 * j + 3], th);
        }
        const uint2 sp = lds_u64_a(sbase + i * 64 + gq * 8);
        const float S = __half2float(__ushort_as_half(static_cast<unsigned short>(q < 2 ? (sp.x >> (16 * q)) : (sp.y >> (16 * (q - 2))))));
        const float zq = 3.f;
        acc[q] = fmaf(S, fmaf(fmaf(th, 0.0625f, tl), 16777216.f, -zq * xsum[g * 4 + t]), acc[q]);
      }
    }
  }
  unsigned long long c1 = clock64();
  float s = 0;
  for (int e = 0; e < 8; ++e) s += acc[e] + Dk[e / 4][e % 4];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (lane == 0) cyc[blockIdx.x * 32 + warp] = c1 - c0;
}
int main() {
  float* o; unsigned long long* cyc; cudaMalloc(&o, 1 << 22); cudaMalloc(&cyc, 8 * 148 * 32);
  const int smem = 65536 + 8192 + 2048 + 512 + 1024;
  const int ntiles = 15 * 64;
  for (int v = 0; v < 4; ++v) {
    for (int nw = 8; nw <= 15; nw += 7) {
      unsigned long long h[32];
      for (int rep = 0; rep < 2; ++rep) {
        if (v == 0) { cudaFuncSetAttribute(ktile<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); ktile<0><<<148, nw * 32, smem>>>(o, cyc, ntiles); }
        if (v == 1) { cudaFuncSetAttribute(ktile<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); ktile<1><<<148, nw * 32, smem>>>(o, cyc, ntiles); }
        if (v == 2) { cudaFuncSetAttribute(ktile<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); ktile<2><<<148, nw * 32, smem>>>(o, cyc, ntiles); }
        if (v == 3) { cudaFuncSetAttribute(ktile<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); ktile<3><<<148, nw * 32, smem>>>(o, cyc, ntiles); }
        cudaDeviceSynchronize();
      }
      cudaMemcpy(h, cyc, 8 * 32, cudaMemcpyDeviceToHost);
      unsigned long long mx = 0; for (int w = 0; w < nw; ++w) mx = h[w] > mx ? h[w] : mx;
      printf("variant %d warps %d: %.0f cycles per tile per warp, %.1f weights/clk/SM  (%s)\n", v, nw, mx / (double)(ntiles / nw),
             ntiles * 4096.0 / mx, cudaGetErrorString(cudaGetLastError()));
    }
  }
}
