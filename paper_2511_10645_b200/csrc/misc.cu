// misc.cu -- standalone activation transform (prefill pre-stage / microbenchmark),
// on-the-fly transform preparation, logical unpack (tests), all-gather permute.
#include <algorithm>
#include <cstdint>
#include <map>
#include <mutex>
#include <tuple>

#include "paro_internal.h"
#include "ptx.cuh"
#include "umma.cuh"
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
#ifndef PARO_TOK_LOCK
#define PARO_TOK_LOCK 8
#endif
constexpr int TOK_LOCK = PARO_TOK_LOCK;  // tokens rotated in lockstep (independent shared-memory chains)

// x' = R_L ... R_1 diag(s) x per (token, group); Eq. 5 in column form,
// the scale first.  One warp = one group x TOK tokens (TOK_LOCK = 8 for activations, 4 for the M build), all
// them in lockstep; the rotation parameters of the group (L <= 8 rotations x 2 slots per
// lane) stay in registers ("the rotation parameters ... fit into registers"),
// the 128 activations of each token of the group in shared memory.  The rotations are
// shared-memory bound (4 loads + 4 stores per lane per rotation); the lockstep tokens give
// the pipe independent work instead of one dependent chain.
template <int TOK>
__global__ void __launch_bounds__(256) transform_kernel(const void* __restrict__ x, int x_bf16, int64_t B, int64_t K,
                                                        int L, const float* __restrict__ svec,
                                                        const float2* __restrict__ rot_cs,
                                                        const uchar2* __restrict__ rot_idx, int rotate,
                                                        __half* __restrict__ xo, int pdl, int prefill_order,
                                                        int identity) {
  __shared__ float scr_all[8][TOK][TGRP];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = static_cast<int>(K / TGRP);
  const int64_t item = static_cast<int64_t>(blockIdx.x) * 8 + warp;  // (token tile, group)
  const int gam = static_cast<int>(item % G);
  const int64_t b0 = (item / G) * TOK;
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
  for (int64_t bc = b0; bc < b0 + TOK && bc < B; bc += TOK) {
    uint2 xv[TOK];
#pragma unroll
    for (int tb = 0; tb < TOK; ++tb) {
      const int64_t b = bc + tb;
      if (TOK >= 4 && identity) {  // (the identity build always runs with 4 or 8 tokens per warp)  // token b = the unit vector e_b of every group (fp16 1.0 = 0x3C00; x_bf16 is 0)
        const int64_t o = b - 4 * lane;
        xv[tb] = make_uint2(o == 0 ? 0x3C00u : o == 1 ? 0x3C000000u : 0u, o == 2 ? 0x3C00u : o == 3 ? 0x3C000000u : 0u);
      } else {
        xv[tb] = (b < B && b < b0 + TOK)
                     ? __ldg(reinterpret_cast<const uint2*>(static_cast<const uint8_t*>(x) +
                                                            (b * K + static_cast<int64_t>(gam) * TGRP + 4 * lane) * 2))
                     : make_uint2(0u, 0u);
      }
    }
#pragma unroll
    for (int tb = 0; tb < TOK; ++tb) {
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
      for (int tb = 0; tb < TOK; ++tb) {
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
    if (TOK >= 4 && identity) {  // (the identity build always runs with 4 or 8 tokens per warp)
      // M^T rows for the dense form: mT[gamma 128 + p][j] = fp16(M_gamma[p][j]) (K-major B operand);
      // the TOK lockstep tokens are the unit vectors e_bc .. e_bc+TOK-1: one 2 TOK-byte store per p
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        uint32_t w[TOK >= 4 ? TOK / 2 : 2];
#pragma unroll
        for (int h = 0; h < (TOK >= 4 ? TOK / 2 : 0); ++h) {
          const __half2 v = __floats2half2_rn(scr_all[warp][2 * h][src[e]], scr_all[warp][2 * h + 1][src[e]]);
          w[h] = *reinterpret_cast<const uint32_t*>(&v);
        }
        __half* o = xo + (static_cast<int64_t>(gam) * TGRP + 4 * lane + e) * TGRP + bc;
        if constexpr (TOK == 8)
          *reinterpret_cast<uint4*>(o) = make_uint4(w[0], w[1], w[2], w[3]);
        else
          *reinterpret_cast<uint2*>(o) = make_uint2(w[0], w[1]);
      }
      __syncwarp();
      continue;
    }
#pragma unroll
    for (int tb = 0; tb < TOK; ++tb) {
      const int64_t b = bc + tb;
      const float* scr = scr_all[warp][tb];
      const __half2 h01 = __floats2half2_rn(scr[src[0]], scr[src[1]]);
      const __half2 h23 = __floats2half2_rn(scr[src[2]], scr[src[3]]);
      uint2 pk;
      pk.x = *reinterpret_cast<const uint32_t*>(&h01);
      pk.y = *reinterpret_cast<const uint32_t*>(&h23);
      if (b < B && b < b0 + TOK)
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
  // tokens per warp: eight in lockstep for many tokens; fewer tokens (decode-sized calls) take one
  // per warp -- the lockstep slots past B would rotate zeros through shared memory for nothing
  const int tok = B >= TOK_LOCK ? TOK_LOCK : 1;
  const int64_t items = ((B + tok - 1) / tok) * G;
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
  return cudaLaunchKernelEx(&cfg, tok == 1 ? transform_kernel<1> : transform_kernel<TOK_LOCK>, x, x_bf16, B, K, L, svec,
                            rot_cs, rot_idx, rotate, static_cast<__half*>(x_out), pdl, prefill_order, 0);
}

// ---------------------------------------------------------------- dense form of the transform (many tokens)
// Per group the transform is one fixed linear map x'_g = M_g x_g with M_g = P R_L ... R_1 diag(s_g)
// (Eq. 5 with the scale first; P the output channel order), a 128 x 128
// matrix.  For many tokens (prefill) applying M_g as a dense contraction on the 5th-generation
// tensor cores replaces eight shared-memory-bound Givens passes (~9 KB of shared-memory traffic
// per token and group) by one 128 x 128 x 128 MMA per 128 tokens, and the transform becomes
// HBM-bound.  M_g is built per call by transform_kernel itself (the same cos/sin/pair tables and
// fp32 Givens arithmetic) applied to the 128 unit vectors: mT[g 128 + p][j] = fp16(M_g[p][j]); the
// contraction rounds M to fp16 (2^-11 relative, the precision of the fp16 x' the GEMM consumes
// anyway) and accumulates in fp32 (TMEM).
//
// CTA = one group x a run of 128-token tiles.  warp 0: TMA producer (M^T once, x tiles into two
// buffers, 128-byte swizzle); warp 1: TMEM allocator + MMA issuer (M = 128 tokens, N = 128
// outputs, K = 16 x 8) into two TMEM accumulators; warps 2..5: epilogue (tcgen05.ld, fp16,
// 16-byte stores: thread = token row).
constexpr int DX_TILE_BYTES = 128 * 128 * 2;             // 32 KB: one operand tile (two 64-wide SW128 boxes)
constexpr int DX_SMEM = 1024 + 3 * DX_TILE_BYTES + 256;  // M^T + two x tiles + barriers (1024-byte aligned)

__global__ void __launch_bounds__(192, 1) transform_dense_kernel(const __grid_constant__ CUtensorMap tmap_x,
                                                                 const __grid_constant__ CUtensorMap tmap_m,
                                                                 const __grid_constant__ CUtensorMap tmap_o, int64_t T,
                                                                 int64_t K, __half* __restrict__ xo, int tiles_per_cta,
                                                                 int pdl) {
  extern __shared__ uint8_t dsm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* m_s = sm;                        // M^T [128 p][128 j]: two [128][64] SW128 boxes
  uint8_t* x_s = sm + DX_TILE_BYTES;        // [2][128 tokens][128 j]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 3 * DX_TILE_BYTES);
  uint64_t* m_full = bar;                   // 1
  uint64_t* x_full = bar + 1;               // 2
  uint64_t* x_empty = bar + 3;              // 2
  uint64_t* acc_full = bar + 5;             // 2
  uint64_t* acc_empty = bar + 7;            // 2
  uint32_t* tmem_sh = reinterpret_cast<uint32_t*>(bar + 9);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = static_cast<int>(blockIdx.y);
  const int64_t n_tiles = (T + 127) / 128;
  const int64_t tile0 = static_cast<int64_t>(blockIdx.x) * tiles_per_cta;
  const int64_t tile_end = n_tiles < tile0 + tiles_per_cta ? n_tiles : tile0 + tiles_per_cta;
  const int nt = tile_end > tile0 ? static_cast<int>(tile_end - tile0) : 0;
  if (threadIdx.x == 0) {
    mbar_init(m_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&x_full[i], 1);
      mbar_init(&x_empty[i], 1);
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 128);
    }
    fence_mbar_init();
    prefetch_tmap(&tmap_x);
    prefetch_tmap(&tmap_m);
    prefetch_tmap(&tmap_o);
  }
  if (warp == 1) tmem_alloc(tmem_sh, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_sh;
  if (pdl) pdl_wait();  // M^T (previous kernel) and x (the kernel before it) are complete
  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(m_full, DX_TILE_BYTES);
      tma_load_2d(m_s, &tmap_m, 0, g * 128, m_full);
      tma_load_2d(m_s + DX_TILE_BYTES / 2, &tmap_m, 64, g * 128, m_full);
      for (int i = 0; i < nt; ++i) {
        const int b = i & 1;
        mbar_wait(&x_empty[b], ((i >> 1) & 1) ^ 1);
        uint8_t* dst = x_s + b * DX_TILE_BYTES;
        const int row = static_cast<int>((tile0 + i) * 128);
        mbar_arrive_expect_tx(&x_full[b], DX_TILE_BYTES);
        tma_load_2d(dst, &tmap_x, g * 128, row, &x_full[b]);
        tma_load_2d(dst + DX_TILE_BYTES / 2, &tmap_x, g * 128 + 64, row, &x_full[b]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_f16_f32(128, 128);
      mbar_wait(m_full, 0);
      const uint64_t mdesc = smem_desc_sw128(m_s);
      for (int i = 0; i < nt; ++i) {
        const int b = i & 1;
        mbar_wait(&acc_empty[b], ((i >> 1) & 1) ^ 1);
        mbar_wait(&x_full[b], (i >> 1) & 1);
        tc_fence_after();
        const uint64_t xdesc = smem_desc_sw128(x_s + b * DX_TILE_BYTES);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // K = 16 per MMA: 32 bytes within a 64-wide box, box 1 for kk >= 4
          const uint64_t koff = static_cast<uint64_t>((kk >> 2) * (DX_TILE_BYTES / 2 / 16) + (kk & 3) * 2);
          mma_f16_ss(tbase + b * 128, xdesc + koff, mdesc + koff, idesc, kk > 0 ? 1u : 0u);
        }
        mma_commit(&acc_full[b]);  // (x_empty: the epilogue, once its store has read the buffer)
      }
    }
  } else {
    // epilogue: warp w reads TMEM lanes 32 (w % 4) .. + 31 = token rows of the tile, rounds to
    // fp16 and writes them into the tile's x buffer (the MMA has consumed it) in the same 128-byte
    // swizzled layout; one thread then stores the tile with TMA (rows past T are clipped) and
    // releases the buffer to the producer once the store has read it
    const int q = warp & 3, r = q * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    for (int i = 0; i < nt; ++i) {
      const int b = i & 1;
      uint8_t* stg = x_s + b * DX_TILE_BYTES;
      mbar_wait(&acc_full[b], (i >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int cb = 0; cb < 4; ++cb) {
        uint32_t v[32];
        tmem_ld32(tbase + b * 128 + cb * 32 + lane_off, v);
        tmem_ld_wait();
        if (cb == 3) {
          tc_fence_before();
          mbar_arrive(&acc_empty[b]);
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {  // 16-byte chunk cc = 4 cb + e of the row: box cc / 8, swizzled
          uint32_t h[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const __half2 p2 = __floats2half2_rn(__uint_as_float(v[8 * e + 2 * k]), __uint_as_float(v[8 * e + 2 * k + 1]));
            h[k] = *reinterpret_cast<const uint32_t*>(&p2);
          }
          const int cc = 4 * cb + e;
          *reinterpret_cast<uint4*>(stg + (cc >> 3) * (DX_TILE_BYTES / 2) + r * 128 + (((cc & 7) ^ (r & 7)) << 4)) =
              make_uint4(h[0], h[1], h[2], h[3]);
        }
      }
      fence_async_smem();          // my writes -> the TMA engine
      named_bar_sync(1, 128);      // every row of the tile is staged
      if (warp == 2 && lane == 0) {
        const int row = static_cast<int>((tile0 + i) * 128);
        tma_store_2d(&tmap_o, stg, g * 128, row);
        tma_store_2d(&tmap_o, stg + DX_TILE_BYTES / 2, g * 128 + 64, row);
        bulk_commit();
        bulk_wait_read0();
        mbar_arrive(&x_empty[b]);
      }
    }
    if (warp == 2 && lane == 0) bulk_wait0();  // the stores are complete before the grid completes
  }
  tc_fence_before();
  __syncthreads();
  if (pdl) pdl_launch_dependents();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tbase, 256);
  }
}

size_t transform_dense_ws_bytes(int64_t K) { return static_cast<size_t>(128 * K * 2); }

cudaError_t launch_transform_dense(const void* x, int x_bf16, int64_t B, int64_t K, int L, const float* svec,
                                   const float2* rot_cs, const uchar2* rot_idx, void* x_out, void* mrows_ws, int pdl,
                                   int prefill_order, cudaStream_t st) {
  const int64_t G = K / TGRP;
  // 1) M rows: transform_kernel on the 128 unit vectors (its PDL wait keeps the dependency on the
  //    kernel before it transitive for the contraction below)
  {
    // four unit vectors per warp up to K = 8192 (32 warps per group spread the build over the SMs;
    // measured cold: K = 4096 5.8 vs 7.1 us), eight beyond (K = 16384: 10.7 vs 12.8 us)
    const int tok = G <= 64 ? 4 : 8;
    const int64_t items = (128 / tok) * G;
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
    cudaError_t e = cudaLaunchKernelEx(&cfg, tok == 4 ? transform_kernel<4> : transform_kernel<8>,
                                       static_cast<const void*>(nullptr), 0,
                                       static_cast<int64_t>(128), K, L, svec, rot_cs, rot_idx, 1,
                                       static_cast<__half*>(mrows_ws), pdl, prefill_order, 1);
    if (e != cudaSuccess) return e;
  }
  // 2) the contraction
  CUtensorMap tx, tm, to;
  if (x_bf16) return cudaErrorInvalidValue;  // the caller converts bf16 x first (x is read by TMA as fp16)
  if (!make_tmap_2d_f16_sw128(&tx, x, static_cast<uint64_t>(K), static_cast<uint64_t>(B), 64, 128) ||
      !make_tmap_2d_f16_sw128(&tm, mrows_ws, 128, static_cast<uint64_t>(K), 64, 128) ||
      !make_tmap_2d_f16_sw128(&to, x_out, static_cast<uint64_t>(K), static_cast<uint64_t>(B), 64, 128))
    return cudaErrorInvalidValue;
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(transform_dense_kernel), DX_SMEM);
  if (e != cudaSuccess) return e;
  // token tiles per CTA: about two CTAs per SM (96 KB of shared memory and 256 TMEM columns each)
  const int64_t n_tiles = (B + 127) / 128;
  const int64_t want = std::max<int64_t>(1, 2 * device_sm_count() / std::max<int64_t>(1, G));
  const int tpc = static_cast<int>((n_tiles + want - 1) / want);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>((n_tiles + tpc - 1) / tpc), static_cast<unsigned>(G));
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = DX_SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;  // always PDL-chained to the M build (its wait is in the kernel)
  return cudaLaunchKernelEx(&cfg, transform_dense_kernel, tx, tm, to, B, K, static_cast<__half*>(x_out), tpc, 1);
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

namespace paro {
// ---------------------------------------------------------------- SM-driven copy (serving loop I/O)
// dst <- src, 16-byte chunks, grid-stride; either side may be pinned host memory (unified
// addressing: reads / posted writes over PCIe by the SMs instead of a DMA-engine copy node).  Under
// PDL the source is read only after the previous kernel completed, and the next kernel may launch
// (and prefetch) at once.
__global__ void __launch_bounds__(256) copy16_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src, int64_t n16,
                                                     int pdl) {
  if (pdl) {
    pdl_launch_dependents();
    pdl_wait();
  }
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n16;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

cudaError_t launch_copy16(void* dst, const void* src, size_t bytes, int pdl, cudaStream_t st) {
  const int64_t n16 = static_cast<int64_t>(bytes / 16);
  // one 16-byte chunk per thread up to a wave of 148 x 256 threads (PCIe latency-bound: many in flight)
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((n16 + 255) / 256, device_sm_count()));
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
  return cudaLaunchKernelEx(&cfg, copy16_kernel, static_cast<uint4*>(dst), static_cast<const uint4*>(src), n16, pdl);
}
}  // namespace paro
