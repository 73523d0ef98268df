// misc.cu -- standalone activation transform (prefill pre-stage / microbenchmark),
// on-the-fly transform preparation, logical unpack (tests), all-gather permute.
#include <algorithm>
#include <cstdint>
#include <map>
#include <mutex>
#include <tuple>

#include "paro_internal.h"
#include "ptx.cuh"
#include "tile_layout.cuh"

namespace paro {

// ---------------------------------------------------------------- per-device host caches
// Every cached device property / function attribute is keyed by the CURRENT device ordinal
// (cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is a per-device setting) and guarded by
// one mutex, so several host threads and several GPUs in one process are safe.
namespace {
std::mutex g_cache_mu;
std::map<int, int> g_sm_count, g_optin;
std::map<std::pair<int, const void*>, int> g_smem_attr;
std::map<std::tuple<int, const void*, int, int, int>, int> g_int_cache;
int current_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess) {
    cudaGetLastError();
    d = 0;
  }
  return d;
}
}  // namespace

int device_sm_count() {
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(g_cache_mu);
  auto it = g_sm_count.find(dev);
  if (it != g_sm_count.end()) return it->second;
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  if (v <= 0) v = 148;
  g_sm_count[dev] = v;
  return v;
}

int device_smem_optin() {
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(g_cache_mu);
  auto it = g_optin.find(dev);
  if (it != g_optin.end()) return it->second;
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (v <= 0) v = 227 * 1024;
  g_optin[dev] = v;
  return v;
}

cudaError_t ensure_smem_attr(const void* fn, int bytes) {
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(g_cache_mu);
  int& have = g_smem_attr[{dev, fn}];
  if (bytes <= have) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}

int cached_device_int(const void* fn, int a, int b, int c, int (*compute)(const void*, int, int, int)) {
  const int dev = current_device();
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_int_cache.find({dev, fn, a, b, c});
    if (it != g_int_cache.end()) return it->second;
  }
  const int v = compute(fn, a, b, c);  // may call ensure_smem_attr (takes the lock)
  std::lock_guard<std::mutex> lk(g_cache_mu);
  g_int_cache[{dev, fn, a, b, c}] = v;
  return v;
}

constexpr int TGRP = 128;
#ifndef PARO_TOK_PER_WARP
#define PARO_TOK_PER_WARP 8
#endif
#ifndef PARO_TOK_LOCK
#define PARO_TOK_LOCK 8
#endif
constexpr int TOK_PER_WARP = PARO_TOK_PER_WARP;
constexpr int TOK_LOCK = PARO_TOK_LOCK;  // tokens rotated in lockstep (independent shared-memory chains)

// x' = R_L ... R_1 diag(s) x per (token, group); Eq. 5 in column form,
// the scale first.  One warp = one group x TOK_PER_WARP tokens, TOK_LOCK of
// them in lockstep; the rotation parameters of the group (L <= 8 rotations x 2 slots per
// lane) stay in registers ("the rotation parameters ... fit into registers"),
// the 128 activations of each token of the group in shared memory.  The rotations are
// shared-memory bound (4 loads + 4 stores per lane per rotation); the lockstep tokens give
// the pipe independent work instead of one dependent chain.
__global__ void __launch_bounds__(256) transform_kernel(const void* __restrict__ x, int x_bf16, int64_t B, int64_t K,
                                                        int L, const float* __restrict__ svec,
                                                        const float2* __restrict__ rot_cs,
                                                        const uchar2* __restrict__ rot_idx, int rotate,
                                                        __half* __restrict__ xo, int pdl, int prefill_order,
                                                        int identity) {
  __shared__ float scr_all[8][TOK_LOCK][TGRP];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = static_cast<int>(K / TGRP);
  const int64_t item = static_cast<int64_t>(blockIdx.x) * 8 + warp;  // (token tile, group)
  const int gam = static_cast<int>(item % G);
  const int64_t b0 = (item / G) * TOK_PER_WARP;
  if (b0 >= B) return;
  // records [G][L][32 lanes]: (cos0, sin0, cos1, sin1) / (i0, j0, i1, j1) of slots l and
  // l + 32 of rotation t
  float4 csr[8];
  uint32_t ixr[8];
  const int Le = rotate ? L : 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    if (t < Le) {
      const int64_t rec = (static_cast<int64_t>(gam) * L + t) * 32 + lane;
      csr[t] = __ldg(reinterpret_cast<const float4*>(rot_cs) + rec);
      ixr[t] = __ldg(reinterpret_cast<const uint32_t*>(rot_idx) + rec);
    }
  }
  const float4 sv = rotate ? __ldg(reinterpret_cast<const float4*>(svec + gam * TGRP) + lane)
                           : make_float4(1.f, 1.f, 1.f, 1.f);
  // identity mode reads no activations: it runs under the previous kernel and waits for it only
  // before exiting (so a PDL dependent of this kernel still sees the previous kernel complete)
  if (pdl && !identity) pdl_wait();
  // output position p of the group: natural (channel p) or prefill order (channel prefill_channel(p))
  int src[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) src[e] = prefill_order ? prefill_channel(4 * lane + e) : 4 * lane + e;
  for (int64_t bc = b0; bc < b0 + TOK_PER_WARP && bc < B; bc += TOK_LOCK) {
    uint2 xv[TOK_LOCK];
#pragma unroll
    for (int tb = 0; tb < TOK_LOCK; ++tb) {
      const int64_t b = bc + tb;
      if (identity) {  // token b = the unit vector e_b of every group (fp16 1.0 = 0x3C00; x_bf16 is 0)
        const int64_t o = b - 4 * lane;
        xv[tb] = make_uint2(o == 0 ? 0x3C00u : o == 1 ? 0x3C000000u : 0u, o == 2 ? 0x3C00u : o == 3 ? 0x3C000000u : 0u);
      } else {
        xv[tb] = (b < B && b < b0 + TOK_PER_WARP)
                     ? __ldg(reinterpret_cast<const uint2*>(static_cast<const uint8_t*>(x) +
                                                            (b * K + static_cast<int64_t>(gam) * TGRP + 4 * lane) * 2))
                     : make_uint2(0u, 0u);
      }
    }
#pragma unroll
    for (int tb = 0; tb < TOK_LOCK; ++tb) {
      float2 f01, f23;
      if (x_bf16) {
        f01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xv[tb].x));
        f23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xv[tb].y));
      } else {
        f01 = __half22float2(*reinterpret_cast<const __half2*>(&xv[tb].x));
        f23 = __half22float2(*reinterpret_cast<const __half2*>(&xv[tb].y));
      }
      *reinterpret_cast<float4*>(&scr_all[warp][tb][4 * lane]) =
          make_float4(f01.x * sv.x, f01.y * sv.y, f23.x * sv.z, f23.y * sv.w);
    }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      if (t >= Le) break;
      const uint32_t i0 = ixr[t] & 0xff, j0 = (ixr[t] >> 8) & 0xff;
      const uint32_t i1 = (ixr[t] >> 16) & 0xff, j1 = ixr[t] >> 24;
#pragma unroll
      for (int tb = 0; tb < TOK_LOCK; ++tb) {
        float* scr = scr_all[warp][tb];
        const float a0 = scr[i0], c0 = scr[j0];
        const float a1 = scr[i1], c1 = scr[j1];
        scr[i0] = csr[t].x * a0 - csr[t].y * c0;
        scr[j0] = csr[t].y * a0 + csr[t].x * c0;
        scr[i1] = csr[t].z * a1 - csr[t].w * c1;
        scr[j1] = csr[t].w * a1 + csr[t].z * c1;
      }
      __syncwarp();
    }
#pragma unroll
    for (int tb = 0; tb < TOK_LOCK; ++tb) {
      const int64_t b = bc + tb;
      const float* scr = scr_all[warp][tb];
      const __half2 h01 = __floats2half2_rn(scr[src[0]], scr[src[1]]);
      const __half2 h23 = __floats2half2_rn(scr[src[2]], scr[src[3]]);
      uint2 pk;
      pk.x = *reinterpret_cast<const uint32_t*>(&h01);
      pk.y = *reinterpret_cast<const uint32_t*>(&h23);
      if (b < B && b < b0 + TOK_PER_WARP)
        *reinterpret_cast<uint2*>(xo + b * K + static_cast<int64_t>(gam) * TGRP + 4 * lane) = pk;
    }
    __syncwarp();
  }
  if (pdl && identity) pdl_wait();
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
                            static_cast<__half*>(x_out), pdl, prefill_order, 0);
}

// ---------------------------------------------------------------- dense form of the transform (many tokens)
// Per group the transform is one fixed linear map x'_g = M_g x_g with M_g = P R_L ... R_1 diag(s_g)
// (Eq. 5 with the scale first; P the output channel order), a 128 x 128
// matrix.  For many tokens (prefill) applying M_g as a dense contraction on the tensor cores moves
// ~2 KB of shared memory per (token, group) instead of the ~9 KB of eight Givens passes, so the
// transform becomes HBM-bound.  M_g is built per call by transform_kernel itself (the same
// cos/sin/pair tables, the same fp32 Givens arithmetic) applied to the 128 unit vectors e_j:
// mrows[j][g 128 + p] = fp16(M_g[p][j]); the contraction then rounds M to fp16 (2^-11 relative,
// the precision of the fp16 x' the GEMM consumes anyway) and accumulates in fp32.
constexpr int DX_ROW = 136;  // padded fp16 row (272 B): conflict-free ldmatrix rows and epilogue writes
constexpr int DX_SMEM = 3 * 128 * DX_ROW * 2;  // M + two token tiles

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void hmma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                          uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// One CTA = one group x a run of 128-token tiles: the group's M rows are staged once, the token
// tiles stream through two shared-memory buffers (cp.async of tile i + 1 overlaps the MMAs of
// tile i).  Warp w: tokens 16 w .. 16 w + 15 of a tile, all 128 outputs (16 m16n8k16 n-tiles x 8
// k-steps); its result is staged back over its own input rows and stored with 16-byte stores.
// bf16 x is converted to fp16 in shared memory (exact in fp16's normal range).
__global__ void __launch_bounds__(256, 2) transform_dense_kernel(const void* __restrict__ x, int x_bf16, int64_t T,
                                                              int64_t K, const __half* __restrict__ mrows,
                                                              __half* __restrict__ xo, int tiles_per_cta, int pdl) {
  extern __shared__ __align__(16) uint8_t dsm[];
  __half* ms = reinterpret_cast<__half*>(dsm);  // [128 inputs j][DX_ROW]: M_g^T, row j = image of e_j
  __half* const xb0 = ms + 128 * DX_ROW;  // [2][128 tokens][DX_ROW]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int64_t c0 = static_cast<int64_t>(blockIdx.y) * TGRP;
  const int64_t n_tiles = (T + 127) / 128;
  const int64_t tile0 = static_cast<int64_t>(blockIdx.x) * tiles_per_cta;
  const int64_t tile1 = min(n_tiles, tile0 + tiles_per_cta);
  if (pdl) pdl_wait();  // M (previous kernel) and x (the kernel before it) are complete
  auto load_x = [&](int64_t tile, __half* dst) {  // 2048 16-byte chunks; rows past T are zero
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const int c = it * 256 + tid, r = c >> 4, q = c & 15;
      const int64_t t = tile * 128 + r;
      if (t < T)
        cp_async16(dst + r * DX_ROW + 8 * q, static_cast<const uint8_t*>(x) + (t * K + c0 + 8 * q) * 2);
      else
        *reinterpret_cast<uint4*>(dst + r * DX_ROW + 8 * q) = make_uint4(0u, 0u, 0u, 0u);
    }
  };
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const int c = it * 256 + tid, r = c >> 4, q = c & 15;
    cp_async16(ms + r * DX_ROW + 8 * q, mrows + static_cast<int64_t>(r) * K + c0 + 8 * q);
  }
  if (tile0 < tile1) load_x(tile0, xb0);
  cp_async_commit();
  const uint32_t xa_off = ((16 * warp + (lane & 15)) * DX_ROW + ((lane >> 4) << 3)) * 2;
  const uint32_t mb = smem_u32(ms + ((lane & 7) + (((lane >> 3) & 1) << 3)) * DX_ROW + ((lane >> 4) << 3));
  const int gq = lane >> 2, tq = lane & 3;
#pragma unroll 1
  for (int64_t tile = tile0; tile < tile1; ++tile) {
    const int b = static_cast<int>(tile - tile0) & 1;
    __half* xs = xb0 + b * (128 * DX_ROW);
    if (tile + 1 < tile1) load_x(tile + 1, xb0 + (b ^ 1) * (128 * DX_ROW));  // released by the barrier below
    cp_async_commit();
    cp_async_wait<1>();  // this tile (and M) landed
    if (x_bf16) {  // my own chunks, in place
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const int c = it * 256 + tid, r = c >> 4, q = c & 15;
        uint4* pv = reinterpret_cast<uint4*>(xs + r * DX_ROW + 8 * q);
        uint4 v = *pv;
        uint32_t* w = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
          const __half2 h = __floats2half2_rn(f.x, f.y);
          w[e] = *reinterpret_cast<const uint32_t*>(&h);
        }
        *pv = v;
      }
    }
    __syncthreads();
    float acc[16][4];
#pragma unroll
    for (int n = 0; n < 16; ++n) acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;
    const uint32_t xa = smem_u32(xs) + xa_off;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      uint32_t a0, a1, a2, a3;
      ldsm_x4(xa + kk * 32, a0, a1, a2, a3);
#pragma unroll
      for (int i = 0; i < 8; ++i) {  // n-tiles 2 i, 2 i + 1
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(mb + (16 * kk * DX_ROW + 16 * i) * 2, b0, b1, b2, b3);
        hmma16816(acc[2 * i], a0, a1, a2, a3, b0, b1);
        hmma16816(acc[2 * i + 1], a0, a1, a2, a3, b2, b3);
      }
    }
    __syncwarp();  // every lane's ldmatrix of this warp's rows is done: reuse them for the output
    __half* orow = xs + (16 * warp + gq) * DX_ROW + 2 * tq;
#pragma unroll
    for (int n = 0; n < 16; ++n) {
      *reinterpret_cast<__half2*>(orow + 8 * n) = __floats2half2_rn(acc[n][0], acc[n][1]);
      *reinterpret_cast<__half2*>(orow + 8 * DX_ROW + 8 * n) = __floats2half2_rn(acc[n][2], acc[n][3]);
    }
    __syncwarp();
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const int c = it * 32 + lane, r = c >> 4, q = c & 15;
      const int64_t t = tile * 128 + 16 * warp + r;
      if (t < T)
        *reinterpret_cast<uint4*>(xo + t * K + c0 + 8 * q) =
            *reinterpret_cast<const uint4*>(xs + (16 * warp + r) * DX_ROW + 8 * q);
    }
    __syncthreads();  // buffer b is free for the load of tile + 2
  }
  cp_async_wait<0>();
  if (pdl) pdl_launch_dependents();
}

size_t transform_dense_ws_bytes(int64_t K) { return static_cast<size_t>(128 * K * 2); }

cudaError_t launch_transform_dense(const void* x, int x_bf16, int64_t B, int64_t K, int L, const float* svec,
                                   const float2* rot_cs, const uchar2* rot_idx, void* x_out, void* mrows_ws, int pdl,
                                   int prefill_order, cudaStream_t st) {
  const int64_t G = K / TGRP;
  // 1) M rows: transform_kernel on the 128 unit vectors (its PDL wait keeps the dependency on the
  //    kernel before it transitive for the contraction below)
  {
    const int64_t items = (128 / TOK_PER_WARP) * G;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>((items + 7) / 8));
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    if (pdl) {
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
    }
    cudaError_t e = cudaLaunchKernelEx(&cfg, transform_kernel, static_cast<const void*>(nullptr), 0,
                                       static_cast<int64_t>(128), K, L, svec, rot_cs, rot_idx, 1,
                                       static_cast<__half*>(mrows_ws), pdl, prefill_order, 1);
    if (e != cudaSuccess) return e;
  }
  // 2) the contraction
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(transform_dense_kernel), DX_SMEM);
  if (e != cudaSuccess) return e;
  // token tiles per CTA: about two CTAs per SM (two fit: 104 KB of shared memory each), at least one
  const int64_t n_tiles = (B + 127) / 128;
  const int64_t want = std::max<int64_t>(1, 2 * device_sm_count() / std::max<int64_t>(1, G));
  const int tpc = static_cast<int>((n_tiles + want - 1) / want);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>((n_tiles + tpc - 1) / tpc), static_cast<unsigned>(G));
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = DX_SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;  // always PDL-chained to the M build (its wait is in the kernel)
  return cudaLaunchKernelEx(&cfg, transform_dense_kernel, x, x_bf16, B, K, static_cast<const __half*>(mrows_ws),
                            static_cast<__half*>(x_out), tpc, 1);
}

// On-the-fly preparation of (cos, sin, i, j) from device theta / pairs (no validation of
// Definition 1: the caller guarantees it).  One 64-thread block per (group, rotation), one
// thread per slot.  An absent slot ((-1, -1) or p >= P) becomes the identity pair (u, u)
// with cos = 1, sin = 0 on the lowest channel u that no present pair of this rotation
// touches: the runtime kernels then read and write only in-range channels, and the
// identity update writes back the value it read (no race with a present pair, whose
// channels are all different from u).  If every slot is present there is no absent slot.
__global__ void __launch_bounds__(64) prepare_transform_kernel(const float* __restrict__ theta,
                                                               const int16_t* __restrict__ pairs, int G, int L, int P,
                                                               float2* __restrict__ rot_cs,
                                                               uchar2* __restrict__ rot_idx) {
  __shared__ uint32_t used[4];
  const int slot = threadIdx.x;
  const int64_t gt = blockIdx.x;  // gamma * L + t
  if (slot < 4) used[slot] = 0u;
  __syncthreads();
  int i = -1, j = -1;
  if (slot < P) {
    const int64_t src = gt * P + slot;
    i = pairs[2 * src];
    j = pairs[2 * src + 1];
    if (i < 0 || j < 0 || i >= 128 || j >= 128) i = j = -1;
  }
  if (i >= 0) {
    atomicOr(&used[i >> 5], 1u << (i & 31));
    atomicOr(&used[j >> 5], 1u << (j & 31));
  }
  __syncthreads();
  float2 cs = make_float2(1.f, 0.f);
  uchar2 ij;
  if (i >= 0) {
    float sn, c;
    sincosf(theta[gt * P + slot], &sn, &c);
    cs = make_float2(c, sn);
    ij = make_uchar2(static_cast<unsigned char>(i), static_cast<unsigned char>(j));
  } else {
    int u = 0;
    for (int w = 0; w < 4; ++w)
      if (~used[w]) {
        u = 32 * w + __ffs(~used[w]) - 1;
        break;
      }
    ij = make_uchar2(static_cast<unsigned char>(u), static_cast<unsigned char>(u));
  }
  const int64_t dst = (gt * 32 + (slot & 31)) * 2 + (slot >> 5);  // [G][L][32][2] record
  rot_cs[dst] = cs;
  rot_idx[dst] = ij;
}

cudaError_t launch_prepare_transform(const float* theta, const int16_t* pairs, int G, int L, int P, float2* rot_cs,
                                     uchar2* rot_idx, cudaStream_t st) {
  const int64_t n = static_cast<int64_t>(G) * L;
  if (n == 0) return cudaSuccess;
  prepare_transform_kernel<<<static_cast<unsigned>(n), 64, 0, st>>>(theta, pairs, G, L, P, rot_cs, rot_idx);
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
