// misc.cu -- standalone activation transform (prefill pre-stage / microbenchmark),
// on-the-fly transform preparation, logical unpack (tests), all-gather permute.
#include <cstdint>

#include "paro_internal.h"
#include "ptx.cuh"
#include "tile_layout.cuh"

namespace paro {

constexpr int TGRP = 128;
constexpr int TOK_PER_WARP = 8;

// x' = R_L ... R_1 diag(s) x per (token, group); Eq. 5 in column form,
// the scale first.  One warp = one group x TOK_PER_WARP tokens; the
// rotation parameters of the group (L <= 8 rotations x 2 slots per lane) stay in
// registers ("the rotation parameters ... fit into registers"), the
// 128 activations of the group in shared memory.
__global__ void __launch_bounds__(256) transform_kernel(const void* __restrict__ x, int x_bf16, int64_t B, int64_t K,
                                                        int L, const float* __restrict__ svec,
                                                        const float2* __restrict__ rot_cs,
                                                        const uchar2* __restrict__ rot_idx, int rotate,
                                                        __half* __restrict__ xo, int pdl, int prefill_order) {
  __shared__ float scr_all[8][132];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* scr = scr_all[warp];
  const int G = static_cast<int>(K / TGRP);
  const int64_t item = static_cast<int64_t>(blockIdx.x) * 8 + warp;  // (token tile, group)
  const int gam = static_cast<int>(item % G);
  const int64_t b0 = (item / G) * TOK_PER_WARP;
  if (b0 >= B) return;
  // records [G][L][32 lanes]: (cos0, sin0, cos1, sin1) / (i0, j0, i1, j1) of slots l and
  // l + 32 of rotation t
  float4 csr[8];
  uint32_t ixr[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    if (t < L && rotate) {
      const int64_t rec = (static_cast<int64_t>(gam) * L + t) * 32 + lane;
      csr[t] = __ldg(reinterpret_cast<const float4*>(rot_cs) + rec);
      ixr[t] = __ldg(reinterpret_cast<const uint32_t*>(rot_idx) + rec);
    } else {
      csr[t] = make_float4(1.f, 0.f, 1.f, 0.f);
      ixr[t] = 0x80808080u;
    }
  }
  float sv[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) sv[i] = rotate ? svec[gam * TGRP + lane + 32 * i] : 1.f;
  if (pdl) pdl_wait();
  for (int64_t b = b0; b < b0 + TOK_PER_WARP && b < B; ++b) {
    const int64_t base = b * K + static_cast<int64_t>(gam) * TGRP;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int k = lane + 32 * i;
      const float v = x_bf16 ? __bfloat162float(static_cast<const __nv_bfloat16*>(x)[base + k])
                             : __half2float(static_cast<const __half*>(x)[base + k]);
      scr[k] = v * sv[i];
    }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      if (t >= L || !rotate) break;
      const uint32_t i0 = ixr[t] & 0xff, j0 = (ixr[t] >> 8) & 0xff;
      const uint32_t i1 = (ixr[t] >> 16) & 0xff, j1 = ixr[t] >> 24;
      const float a0 = scr[i0], c0 = scr[j0];
      const float a1 = scr[i1], c1 = scr[j1];
      scr[i0] = csr[t].x * a0 - csr[t].y * c0;
      scr[j0] = csr[t].y * a0 + csr[t].x * c0;
      scr[i1] = csr[t].z * a1 - csr[t].w * c1;
      scr[j1] = csr[t].w * a1 + csr[t].z * c1;
      __syncwarp();
    }
    // natural order: lane writes channels 4l..4l+3.  prefill_order: position p of the group
    // holds channel prefill_channel(p) (the order the prefill dequantiser emits weights in)
    float v4[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) v4[e] = scr[prefill_order ? prefill_channel(4 * lane + e) : 4 * lane + e];
    const __half2 h01 = __floats2half2_rn(v4[0], v4[1]);
    const __half2 h23 = __floats2half2_rn(v4[2], v4[3]);
    uint2 pk;
    pk.x = *reinterpret_cast<const uint32_t*>(&h01);
    pk.y = *reinterpret_cast<const uint32_t*>(&h23);
    *reinterpret_cast<uint2*>(xo + base + 4 * lane) = pk;
    __syncwarp();
  }
  if (pdl) pdl_launch_dependents();
}

cudaError_t launch_transform(const void* x, int x_bf16, int64_t B, int64_t K, int L, const float* svec,
                             const float2* rot_cs, const uchar2* rot_idx, int rotate, void* x_out, int pdl,
                             int prefill_order, cudaStream_t st) {
  const int64_t G = K / TGRP;
  const int64_t items = ((B + TOK_PER_WARP - 1) / TOK_PER_WARP) * G;
  const int64_t blocks = (items + 7) / 8;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(blocks));
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  if (pdl) {
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  return cudaLaunchKernelEx(&cfg, transform_kernel, x, x_bf16, B, K, L, svec, rot_cs, rot_idx, rotate,
                            static_cast<__half*>(x_out), pdl, prefill_order);
}

// On-the-fly preparation of (cos, sin, i, j) from device theta / pairs (no validation).
__global__ void prepare_transform_kernel(const float* __restrict__ theta, const int16_t* __restrict__ pairs, int G,
                                         int L, int P, float2* __restrict__ rot_cs, uchar2* __restrict__ rot_idx) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;  // (gamma, t, slot<64)
  if (e >= static_cast<int64_t>(G) * L * 64) return;
  const int slot = static_cast<int>(e % 64);
  const int64_t gt = e / 64;
  const int64_t gam = gt / L, t = gt % L;
  const int64_t dst = ((gam * L + t) * 32 + (slot & 31)) * 2 + (slot >> 5);  // [G][L][32][2] record
  float2 cs = make_float2(1.f, 0.f);
  uchar2 ij = make_uchar2(128, 128);
  if (slot < P) {
    const int64_t src = gt * P + slot;
    const int i = pairs[2 * src], j = pairs[2 * src + 1];
    if (i >= 0 && j >= 0 && i < 128 && j < 128) {
      float s, c;
      sincosf(theta[src], &s, &c);
      cs = make_float2(c, s);
      ij = make_uchar2(static_cast<unsigned char>(i), static_cast<unsigned char>(j));
    }
  }
  rot_cs[dst] = cs;
  rot_idx[dst] = ij;
}

cudaError_t launch_prepare_transform(const float* theta, const int16_t* pairs, int G, int L, int P, float2* rot_cs,
                                     uchar2* rot_idx, cudaStream_t st) {
  const int64_t n = static_cast<int64_t>(G) * L * 64;
  if (n == 0) return cudaSuccess;
  prepare_transform_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(theta, pairs, G, L, P, rot_cs,
                                                                                   rot_idx);
  return cudaGetLastError();
}

// tile layout -> logical codes [N][K], scales [N][G] (fp16), zeros [N][G]
__global__ void unpack_kernel(const uint8_t* __restrict__ codes, const __half* __restrict__ scales,
                              const uint8_t* __restrict__ zeros, int64_t N, int64_t K, uint8_t* __restrict__ cu8,
                              __half* __restrict__ sf16, uint8_t* __restrict__ zu8) {
  const int64_t G = K / TGRP;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < N * K; i += stride) {
    const int64_t n = i / K, k = i % K;
    const int64_t T = (n / TILE_ROWS) * G + k / TGRP;
    int byte, hi;
    tile_pos(static_cast<int>(k % TGRP), &byte, &hi);
    const uint8_t b = codes[T * TILE_CODE_BYTES + (n % TILE_ROWS) * 64 + byte];
    cu8[i] = hi ? (b >> 4) : (b & 15);
  }
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < N * G; i += stride) {
    const int64_t n = i / G, g = i % G;
    const int64_t T = (n / TILE_ROWS) * G + g;
    const int r = static_cast<int>(n % TILE_ROWS);
    sf16[i] = scales[T * TILE_ROWS + tile_scale_idx(r)];
    const uint8_t b = zeros[T * TILE_ZERO_BYTES + tile_zero_byte(r)];
    zu8[i] = tile_zero_hi(r) ? (b >> 4) : (b & 15);
  }
}

cudaError_t launch_unpack(const uint8_t* codes, const uint8_t* scales, const uint8_t* zeros, int64_t N, int64_t K,
                          uint8_t* codes_u8, uint8_t* scales_f16, uint8_t* zeros_u8, cudaStream_t st) {
  unpack_kernel<<<1024, 256, 0, st>>>(codes, reinterpret_cast<const __half*>(scales), zeros, N, K, codes_u8,
                                      reinterpret_cast<__half*>(scales_f16), zeros_u8);
  return cudaGetLastError();
}

// [world][B][Ns] (rank-major all-gather result) -> [B][world*Ns]
__global__ void permute_gather_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, int world,
                                      int64_t B, int64_t Ns, int eb) {
  const int64_t tot = static_cast<int64_t>(world) * B * Ns;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < tot;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / (B * Ns), rem = i % (B * Ns), b = rem / Ns, n = rem % Ns;
    const int64_t d = b * (world * Ns) + r * Ns + n;
    for (int e = 0; e < eb; ++e) dst[d * eb + e] = src[i * eb + e];
  }
}

cudaError_t launch_permute_gather(const void* src, void* dst, int world, int64_t B, int64_t Ns, int elem_bytes,
                                  cudaStream_t st) {
  permute_gather_kernel<<<256, 256, 0, st>>>(static_cast<const uint8_t*>(src), static_cast<uint8_t*>(dst), world, B,
                                             Ns, elem_bytes);
  return cudaGetLastError();
}

}  // namespace paro
