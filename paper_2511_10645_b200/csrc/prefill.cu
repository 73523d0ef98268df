// prefill.cu -- prefill path (B > 16 tokens): tcgen05 / TMEM GEMM with an in-kernel
// INT4 -> fp16 dequant producer (epilogue a8).
//
//   y[t, n] = sum_k x'[t, k] * S[n, k/128] * (q[n, k] - z[n, k/128])   (+ bias[n])
//
// Orientation: the WEIGHTS are the MMA's M operand (128 rows per CTA tile) and live in
// TMEM: four dequant warps turn packed nibbles into fp16 (q - z) * S (exact
// subtraction, one rounding in the multiply) and write them with tcgen05.st straight
// into tensor memory -- the A operand of tcgen05.mma may come from TMEM, so the
// dequantised weights never touch shared memory.  The rotated activations x' (fp16,
// produced by the transform pre-stage into an L2-resident workspace) are the N
// operand (256 tokens per tile), loaded by TMA with 128-byte swizzle into a
// shared-memory ring.  One elected thread issues tcgen05.mma (M=128, N=256, K=16)
// into a 128 x 256 fp32 accumulator in TMEM; four epilogue warps read it back with
// tcgen05.ld, add the bias, convert and store y.
//
// Stage ks of a row is the 32-byte half (ks & 1) of its tile-layout row in group ks / 2;
// the dequantiser emits fp16 pairs straight from one AND/OR mask per nibble pair of a
// 32-bit code word (no byte permutes).  The pre-stage stores x' in that same channel
// order (prefill_pos, tile_layout.cuh): one permutation along K on both operands leaves
// the contraction unchanged.
//
// Warp roles (512 threads, persistent over tiles):
//   warp 0: TMA producer (x' tiles)     warp 1: MMA issuer     warp 2: TMEM allocator
//   warps 4-7 / 12-15: dequant -> TMEM (A), even / odd K stages   warps 8-11: epilogue (TMEM -> y)
// (eight dequant warps: with four the INT4 -> fp16 producer limited the MMA rate)
#include <cuda.h>
#include <cuda_fp16.h>

#include <cstdint>
#include <mutex>

#include "paro_internal.h"
#include "ptx.cuh"
#include "umma.cuh"
#include "tile_layout.cuh"

namespace paro {

#ifndef PARO_PF_DEEP
#define PARO_PF_DEEP 1  // dequant loads two iterations ahead (0: one)
#endif
constexpr int PF_BM = 128;    // weight rows per tile (MMA M)
constexpr int PF_BK = 64;     // K per pipeline stage (4 MMAs of K=16)
#ifndef PARO_PF_STAGE_EPI
#define PARO_PF_STAGE_EPI 1  // 16-bit y staged in shared memory (coalesced stores, early TMEM release)
#endif
#ifndef PARO_PF_SX
#define PARO_PF_SX 4
#endif
constexpr int PF_SX = PARO_PF_SX;  // x' shared-memory stages (32 KB each at 256 tokens)
constexpr int PF_SA = 8;      // A (dequantised weight) TMEM stages (32 columns each)
constexpr int PF_ACC_COL = 0;
constexpr int PF_A_COL = 256;
constexpr int PF_TMEM_COLS = 512;
#ifndef PARO_PF_NSETS
#define PARO_PF_NSETS 2  // dequant warp sets (4 warps each) taking K-stages round robin
#endif
constexpr int PF_NSETS = PARO_PF_NSETS;
constexpr int PF_THREADS = 512 + 128 * (PF_NSETS - 2);

struct PrefillArgs {
  const uint8_t* codes;
  const __half* scales;
  const uint8_t* zeros;
  const float* bias;
  void* y;
  int y_dtype;
  int B, N, K;
  int pdl;
  // split-K (few tiles, e.g. k / v): item c = (tile c / 2, K half c % 2), one per CTA; the two
  // halves of a tile are a cluster pair and exchange fp32 partials of each other's tokens in DSMEM
  int split;
};

struct PfItem {
  int tile, kb, ke, half;  // half: K half of a split tile, or -1
};
// the i-th work item of this CTA (false past the last)
template <bool SPLIT>
__device__ __forceinline__ bool pf_item(const PrefillArgs& a, int n_tiles, int n_ks, int i, PfItem& it) {
  if (SPLIT) {
    const int c = static_cast<int>(blockIdx.x);
    if (i > 0 || c >= 2 * n_tiles) return false;
    it.tile = c >> 1;
    it.half = c & 1;
    it.kb = it.half * (n_ks / 2);
    it.ke = it.half ? n_ks : n_ks / 2;
    return true;
  }
  const int tile = static_cast<int>(blockIdx.x) + i * static_cast<int>(gridDim.x);
  if (tile >= n_tiles) return false;
  it.tile = tile;
  it.kb = 0;
  it.ke = n_ks;
  it.half = -1;
  return true;
}

__device__ __forceinline__ uint32_t hsub_hmul(uint32_t v, uint32_t zz, uint32_t ss) {
  __half2 a = *reinterpret_cast<__half2*>(&v);
  __half2 z = *reinterpret_cast<__half2*>(&zz);
  __half2 s = *reinterpret_cast<__half2*>(&ss);
  __half2 r = __hmul2(__hsub2(a, z), s);  // (1024+q) - (1024+z) exact, then one rounding
  return *reinterpret_cast<uint32_t*>(&r);
}

#ifndef PARO_PF_SPLITK
#define PARO_PF_SPLITK 1  // few tiles: split-K halves on two SMs (0: 128-token tiles)
#endif
#ifndef PARO_PF_MMA_SPIN
#define PARO_PF_MMA_SPIN 0  // 1: the MMA issuer polls its stage barriers without the suspend hint
#endif
#ifndef PARO_PF_PROF
#define PARO_PF_PROF 0  // 1: the MMA issuer's wait cycles per CTA (acc_empty, A stage, x' stage, total)
#endif
#if PARO_PF_PROF
__device__ unsigned long long g_pf_prof[1024 * 4];
extern "C" int paro_debug_pf_prof(unsigned long long* host, int n) {
  if (n > 1024 * 4) n = 1024 * 4;
  return static_cast<int>(cudaMemcpyFromSymbol(host, g_pf_prof, sizeof(unsigned long long) * n));
}
#endif

// PF_BN: tokens per tile (MMA N): 256, or 128 when 256-token tiles would leave SMs idle (k / v)
template <int PF_BN, bool SPLIT>
__global__ void __launch_bounds__(PF_THREADS, 1)
    prefill_gemm_kernel(const __grid_constant__ CUtensorMap tmap_x, const PrefillArgs a) {
  constexpr uint32_t PF_X_STAGE_BYTES = PF_BN * PF_BK * 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* xs = smem;  // PF_SX * 32 KB
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + PF_SX * PF_X_STAGE_BYTES);
  uint64_t* x_full = bars;
  uint64_t* x_empty = x_full + PF_SX;
  uint64_t* a_full = x_empty + PF_SX;
  uint64_t* a_empty = a_full + PF_SA;
  uint64_t* acc_full = a_empty + PF_SA;
  uint64_t* acc_empty = acc_full + 1;
  uint64_t* xchg = acc_empty + 1;  // split-K: the partner's partial of my tokens landed (st.async bytes)
  uint32_t* tmem_base_sh = reinterpret_cast<uint32_t*>(xchg + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_row_tiles = a.N / PF_BM;
  const int n_tok_tiles = (a.B + PF_BN - 1) / PF_BN;
  const int n_tiles = n_row_tiles * n_tok_tiles;
  const int n_ks = a.K / PF_BK;

  if (threadIdx.x == 0) {
    for (int i = 0; i < PF_SX; ++i) {
      mbar_init(&x_full[i], 1);
      mbar_init(&x_empty[i], 1);
    }
    for (int i = 0; i < PF_SA; ++i) {
      mbar_init(&a_full[i], 128);
      mbar_init(&a_empty[i], 1);
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, 128);
    mbar_init(xchg, 1);
    // split-K: 128 rows x PF_BN / 2 fp32 of the partner's partial (armed before any byte can land)
    if (SPLIT) mbar_arrive_expect_tx(xchg, PF_BM * (PF_BN / 2) * 4);
    fence_mbar_init();
    prefetch_tmap(&tmap_x);
  }
  if (warp == 2) tmem_alloc(tmem_base_sh, PF_TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_base_sh;
  if (SPLIT) {  // both CTAs of the pair initialised their barriers: DSMEM stores are legal
    cluster_arrive_relaxed();
    cluster_wait();
  }
  // every CTA of this (one-wave, persistent) grid is resident: the next kernel may launch now.
  // Dependents wait (griddepcontrol.wait) before reading y; the next linear's transform-matrix
  // build reads only packed tables, so it runs on the SMs' spare resources under this GEMM.
  if (a.pdl) pdl_launch_dependents();
  if (a.pdl) pdl_wait();  // x' is written by the pre-stage kernel

  if (warp == 0) {
    // ---------------- TMA producer: x' tiles [256 tokens x 64 K] (SW128)
    if (lane == 0) {
      uint32_t it = 0;
      PfItem w;
      for (int item = 0; pf_item<SPLIT>(a, n_tiles, n_ks, item, w); ++item) {
        const int tok0 = (w.tile / n_row_tiles) * PF_BN;
        for (int ks = w.kb; ks < w.ke; ++ks, ++it) {
          const int s = it % PF_SX;
          mbar_wait(&x_empty[s], ((it / PF_SX) & 1) ^ 1);
          mbar_arrive_expect_tx(&x_full[s], PF_X_STAGE_BYTES);
          tma_load_2d(xs + s * PF_X_STAGE_BYTES, &tmap_x, ks * PF_BK, tok0, &x_full[s]);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one thread)
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_f16_f32(PF_BM, PF_BN);
      uint32_t it = 0, tcount = 0;
#if PARO_PF_PROF
      unsigned long long w_acc = 0, w_a = 0, w_x = 0, t_beg = clock64();
#define PF_T0 const unsigned long long _t0 = clock64();
#define PF_T1(v) v += clock64() - _t0;
#else
#define PF_T0
#define PF_T1(v)
#endif
      PfItem w;
      for (int item = 0; pf_item<SPLIT>(a, n_tiles, n_ks, item, w); ++item, ++tcount) {
        {
          PF_T0 mbar_wait(acc_empty, (tcount & 1) ^ 1);
          PF_T1(w_acc)
        }
        tc_fence_after();
        for (int ks = w.kb; ks < w.ke; ++ks, ++it) {
          const int sx = it % PF_SX, sa = it % PF_SA;
          {
            PF_T0 if (PARO_PF_MMA_SPIN) mbar_wait_spin(&a_full[sa], (it / PF_SA) & 1); else mbar_wait(&a_full[sa], (it / PF_SA) & 1);
            PF_T1(w_a)
          }
          {
            PF_T0 if (PARO_PF_MMA_SPIN) mbar_wait_spin(&x_full[sx], (it / PF_SX) & 1); else mbar_wait(&x_full[sx], (it / PF_SX) & 1);
            PF_T1(w_x)
          }
          tc_fence_after();
          const uint64_t bdesc = smem_desc_sw128(xs + sx * PF_X_STAGE_BYTES);
#pragma unroll
          for (int kk = 0; kk < PF_BK / 16; ++kk) {
            mma_f16_ts(tbase + PF_ACC_COL, tbase + PF_A_COL + sa * 32 + kk * 8, bdesc + static_cast<uint64_t>(kk * 2),
                       idesc, (ks > w.kb || kk > 0) ? 1u : 0u);
          }
          mma_commit(&x_empty[sx]);
          mma_commit(&a_empty[sa]);
        }
        mma_commit(acc_full);
      }
#if PARO_PF_PROF
      if (blockIdx.x < 1024) {
        g_pf_prof[blockIdx.x * 4 + 0] = w_acc;
        g_pf_prof[blockIdx.x * 4 + 1] = w_a;
        g_pf_prof[blockIdx.x * 4 + 2] = w_x;
        g_pf_prof[blockIdx.x * 4 + 3] = clock64() - t_beg;
      }
#endif
    }
  } else if ((warp >= 4 && warp < 8) || warp >= 12) {
    // ---------------- dequant producer: weight row r of the tile -> TMEM lane r
    const int par = warp < 8 ? 0 : (warp < 16 ? 1 : 2);  // this dequant warp set (K-stages round robin)
    const int r = (warp & 3) * 32 + lane;
    const uint32_t lane_addr = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const int G = a.K / 128;
    uint32_t it_base = 0;  // K-stage counter at the item's first stage (both parity sets)
    PfItem w;
    for (int item = 0; pf_item<SPLIT>(a, n_tiles, n_ks, item, w); ++item) {
      const int n = (w.tile % n_row_tiles) * PF_BM + r;
      const int rt = n % TILE_ROWS;
      const int64_t T0 = static_cast<int64_t>(n / TILE_ROWS) * G;  // first tile of the row block
      // stage ks = half-row (32 bytes) ks & 1 of tile (row block, ks / 2).  The row's code bytes,
      // scale and zero point of my parity's stages are loaded two iterations (four K-stages) ahead:
      // the dequant chain must never wait on a load's full latency (long-scoreboard stalls)
      const uint8_t* crow = a.codes + T0 * TILE_CODE_BYTES + rt * 64;
      struct Pf {
        uint4 c0, c1;
        uint32_t sz;  // S bits | z << 16
      };
      auto load = [&](int ks) {
        Pf f;
        const int64_t T = T0 + (ks >> 1);
        const uint8_t* cp = crow + static_cast<int64_t>(ks >> 1) * TILE_CODE_BYTES + (ks & 1) * 32;
        f.c0 = __ldg(reinterpret_cast<const uint4*>(cp));
        f.c1 = __ldg(reinterpret_cast<const uint4*>(cp + 16));
        const uint32_t sb = __ldg(reinterpret_cast<const unsigned short*>(a.scales) + T * TILE_ROWS + tile_scale_idx(rt));
        const uint32_t zb = __ldg(a.zeros + T * TILE_ZERO_BYTES + tile_zero_byte(rt));
        f.sz = sb | ((tile_zero_hi(rt) ? (zb >> 4) : (zb & 15u)) << 16);
        return f;
      };
      // my stages of the item: those whose global counter has my parity (n_ks / 2 is even here, so
      // for the default round-robin items this is ks = par, par + 2, ...)
      const int ks0 = w.kb + static_cast<int>((static_cast<uint32_t>(par) + PF_NSETS * 4u - it_base % PF_NSETS) % PF_NSETS);
      const int kend = w.ke;
      if (ks0 >= kend) {
        it_base += static_cast<uint32_t>(w.ke - w.kb);
        continue;
      }
      Pf p1 = load(ks0), p2 = (PARO_PF_DEEP && ks0 + PF_NSETS < kend) ? load(ks0 + PF_NSETS) : p1;
      Pf p3 = (PARO_PF_DEEP > 1 && ks0 + 2 * PF_NSETS < kend) ? load(ks0 + 2 * PF_NSETS) : p2;
      uint32_t ss = 0, zz = 0;
      uint32_t it = it_base + static_cast<uint32_t>(ks0 - w.kb);
      for (int ks = ks0; ks < kend; ks += PF_NSETS, it += PF_NSETS) {
        const Pf cur = p1;
        if (PARO_PF_DEEP > 1) {
          p1 = p2;
          p2 = p3;
          if (ks + 3 * PF_NSETS < kend) p3 = load(ks + 3 * PF_NSETS);
        } else if (PARO_PF_DEEP) {
          p1 = p2;
          if (ks + 2 * PF_NSETS < kend) p2 = load(ks + 2 * PF_NSETS);
        } else if (ks + PF_NSETS < kend) {
          p1 = load(ks + PF_NSETS);
        }
        {
          const uint32_t sbits = cur.sz & 0xffffu, z = cur.sz >> 16;
          ss = sbits | (sbits << 16);
          const uint32_t zh = 0x6400u + z;  // 1024 + z
          zz = zh | (zh << 16);
        }
        const uint4 w0 = cur.c0, w1 = cur.c1;
        uint32_t v[32];
        const uint32_t wd[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          const uint32_t w = wd[m];
          v[4 * m + 0] = hsub_hmul((w & 0x000F000Fu) | 0x64006400u, zz, ss);          // nibbles (0, 4)
          v[4 * m + 1] = hsub_hmul(((w >> 4) & 0x000F000Fu) | 0x64006400u, zz, ss);   // (1, 5)
          v[4 * m + 2] = hsub_hmul(((w >> 8) & 0x000F000Fu) | 0x64006400u, zz, ss);   // (2, 6)
          v[4 * m + 3] = hsub_hmul(((w >> 12) & 0x000F000Fu) | 0x64006400u, zz, ss);  // (3, 7)
        }
        const int sa = it % PF_SA;
        mbar_wait(&a_empty[sa], ((it / PF_SA) & 1) ^ 1);
        tc_fence_after();
        tmem_st32(tbase + lane_addr + PF_A_COL + sa * 32, v);
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&a_full[sa]);
      }
      it_base += static_cast<uint32_t>(w.ke - w.kb);
    }
  } else if (warp >= 8) {
    // ---------------- epilogue: accumulator lane r = weight row, column = token
    const int r = (warp - 8) * 32 + lane;
    const uint32_t lane_addr = static_cast<uint32_t>((warp - 8) * 32) << 16;
    uint32_t tcount = 0;
    PfItem w;
    for (int item = 0; pf_item<SPLIT>(a, n_tiles, n_ks, item, w); ++item, ++tcount) {
      const int tile = w.tile;
      const int n = (tile % n_row_tiles) * PF_BM + r;
      const int tok0 = (tile / n_row_tiles) * PF_BN;
      const float bv = a.bias ? a.bias[n] : 0.f;
      mbar_wait(acc_full, tcount & 1);
      tc_fence_after();
      if (SPLIT) {
        // split-K, the two halves of a tile (a cluster pair) finish it together: half h owns the
        // tokens [128 h, 128 h + 128) of the tile.  Each half sends its partial of the OTHER half's
        // tokens straight into the partner's shared memory (st.async, fp32 [row][128 tokens], 16-byte
        // chunks XOR-swizzled by row), waits for the partner's partial of its own tokens, adds it to
        // its accumulator in a fixed order (half 0's partial + half 1's) and stores y for them.
        constexpr int HT = PF_BN / 2;
        const int h = w.half, mine = h * HT, theirs = (1 - h) * HT;
        uint8_t* rx = smem + PF_SX * PF_X_STAGE_BYTES + 1024;  // [128 rows][HT] fp32 = 64 KB
        const uint32_t partner = cluster_ctarank() ^ 1u;
        const uint32_t rx_remote = mapa(smem_u32(rx), partner), bar_remote = mapa(smem_u32(xchg), partner);
#pragma unroll 1
        for (int c = 0; c < HT / 32; ++c) {
          uint32_t v[32];
          tmem_ld32(tbase + lane_addr + PF_ACC_COL + theirs + c * 32, v);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int ch = c * 8 + e;  // 16-byte chunk of the row
            st_async_v4(rx_remote + static_cast<uint32_t>(r * HT * 4 + ((ch ^ (r & 7)) << 4)),
                        make_uint4(v[4 * e], v[4 * e + 1], v[4 * e + 2], v[4 * e + 3]), bar_remote);
          }
        }
        mbar_wait(xchg, 0);  // the partner's partial of my tokens is in rx
        const int n0 = (tile % n_row_tiles) * PF_BM;
        uint16_t* stg = reinterpret_cast<uint16_t*>(smem);  // my x' stages are free: y staging [HT][128]
#pragma unroll 1
        for (int c = 0; c < HT / 32; ++c) {
          uint32_t v[32];
          tmem_ld32(tbase + lane_addr + PF_ACC_COL + mine + c * 32, v);
          tmem_ld_wait();
          if (c == HT / 32 - 1) {
            tc_fence_before();
            mbar_arrive(acc_empty);
          }
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int ch = c * 8 + e;
            const float4 q = *reinterpret_cast<const float4*>(rx + r * HT * 4 + ((ch ^ (r & 7)) << 4));
            const float p4[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float mv = __uint_as_float(v[4 * e + k]);
              const float o = (h == 0 ? mv + p4[k] : p4[k] + mv) + bv;  // half 0's partial first
              const int t = c * 32 + 4 * e + k;
              if (a.y_dtype == 2) {
                if (tok0 + mine + t < a.B) static_cast<float*>(a.y)[static_cast<int64_t>(tok0 + mine + t) * a.N + n] = o;
              } else {
                stg[t * PF_BM + r] = a.y_dtype == 0 ? __half_as_ushort(__float2half_rn(o))
                                                    : __bfloat16_as_ushort(__float2bfloat16_rn(o));
              }
            }
          }
        }
        if (a.y_dtype != 2) {
          named_bar_sync(7, 128);
#pragma unroll 4
          for (int q = r; q < HT * 16; q += 128) {
            const int tk = q >> 4, c16 = q & 15;
            if (tok0 + mine + tk < a.B)
              *reinterpret_cast<uint4*>(static_cast<uint16_t*>(a.y) + static_cast<int64_t>(tok0 + mine + tk) * a.N +
                                        n0 + 8 * c16) = *reinterpret_cast<const uint4*>(stg + tk * PF_BM + 8 * c16);
          }
        }
        continue;
      }
      if (PARO_PF_STAGE_EPI && a.y_dtype != 2) {
        // 16-bit outputs: accumulator -> shared-memory staging [token][128 rows] (the MMA may start
        // the next tile as soon as TMEM is read), then 16-byte coalesced row stores of y
        uint16_t* stg = reinterpret_cast<uint16_t*>(smem + PF_SX * PF_X_STAGE_BYTES + 1024);
#pragma unroll 1
        for (int c = 0; c < PF_BN / 32; ++c) {
          uint32_t v[32];
          tmem_ld32(tbase + lane_addr + PF_ACC_COL + c * 32, v);
          tmem_ld_wait();
          if (c == PF_BN / 32 - 1) {
            tc_fence_before();
            mbar_arrive(acc_empty);
          }
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float f = __uint_as_float(v[i]) + bv;
            stg[(c * 32 + i) * PF_BM + r] = a.y_dtype == 0 ? __half_as_ushort(__float2half_rn(f))
                                                           : __bfloat16_as_ushort(__float2bfloat16_rn(f));
          }
        }
        named_bar_sync(7, 128);
        const int n0 = (tile % n_row_tiles) * PF_BM;
        const int et = (warp - 8) * 32 + lane;
#pragma unroll 4
        for (int q = et; q < PF_BN * 16; q += 128) {
          const int tk = q >> 4, c16 = q & 15;
          if (tok0 + tk < a.B)
            *reinterpret_cast<uint4*>(static_cast<uint16_t*>(a.y) + static_cast<int64_t>(tok0 + tk) * a.N + n0 + 8 * c16) =
                *reinterpret_cast<const uint4*>(stg + tk * PF_BM + 8 * c16);
        }
        named_bar_sync(7, 128);  // staging free for the next tile
        continue;
      }
#pragma unroll 1
      for (int c = 0; c < PF_BN / 32; ++c) {        uint32_t v[32];
        tmem_ld32(tbase + lane_addr + PF_ACC_COL + c * 32, v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int t = tok0 + c * 32 + i;
          if (t < a.B) {
            const float f = __uint_as_float(v[i]) + bv;
            const int64_t o = static_cast<int64_t>(t) * a.N + n;
            if (a.y_dtype == 0)
              static_cast<__half*>(a.y)[o] = __float2half_rn(f);
            else if (a.y_dtype == 1)
              static_cast<__nv_bfloat16*>(a.y)[o] = __float2bfloat16_rn(f);
            else
              static_cast<float*>(a.y)[o] = f;
          }
        }
      }
      tc_fence_before();
      mbar_arrive(acc_empty);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tbase, PF_TMEM_COLS);
  }
}

// ============================================================================ host
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

bool make_tmap_2d_f16_sw128(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint32_t box_inner,
                            uint32_t box_outer) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t gdim[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
  cuuint64_t gstride[1] = {static_cast<cuuint64_t>(inner) * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), gdim, gstride, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool prefill_supported(int64_t B, int64_t N, int64_t K) {
  return B >= 1 && N % PF_BM == 0 && K % PF_BK == 0 && K >= PF_BK && N <= (int64_t(1) << 30) && B < (1 << 30);
}

template <int PF_BN>
static cudaError_t prefill_launch(const void* xq, int64_t B, const PrefillArgs& a, int64_t N, int pdl,
                                  cudaStream_t st) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return cudaErrorNotSupported;
  CUtensorMap tmap;
  const int64_t K = a.K;
  cuuint64_t gdim[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(B)};
  cuuint64_t gstride[1] = {static_cast<cuuint64_t>(K) * 2};
  cuuint32_t box[2] = {PF_BK, PF_BN};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(xq), gdim, gstride, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  // x' stages + barriers (1 KB) + the epilogue's y staging (PF_BN x 128 16-bit values)
  const size_t smem = 1024 + PF_SX * PF_BN * PF_BK * 2 + 1024 + (PARO_PF_STAGE_EPI ? PF_BN * PF_BM * 2 : 0);
  auto kern = a.split ? prefill_gemm_kernel<PF_BN, true> : prefill_gemm_kernel<PF_BN, false>;
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const int64_t tiles = (N / PF_BM) * ((B + PF_BN - 1) / PF_BN);
  const int grid = a.split ? static_cast<int>(2 * tiles)
                           : static_cast<int>(tiles < device_sm_count() ? tiles : device_sm_count());
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(PF_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (pdl) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (a.split) {  // the two K halves of a tile form a cluster (they exchange partials through DSMEM)
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = 2;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, tmap, a);
}

cudaError_t launch_prefill_gemm(const void* xq, int64_t B, const uint8_t* codes, const uint8_t* scales,
                                const uint8_t* zeros, const float* bias, void* y, int y_dtype, int64_t N, int64_t K,
                                int pdl, cudaStream_t st) {
  PrefillArgs a{codes, reinterpret_cast<const __half*>(scales), zeros, bias, y, y_dtype, static_cast<int>(B),
                static_cast<int>(N), static_cast<int>(K), pdl, 0};
  const int64_t tiles256 = (N / PF_BM) * ((B + 255) / 256);
  // few 256-token tiles (e.g. k / v: 1024 x 4096 at 2048 tokens = 64 tiles): each tile as two K
  // halves on a cluster pair of SMs (every SM busy, each half at N = 256; same-box k_proj 41.8 -> 34.7 us)
  if (PARO_PF_SPLITK && 2 * tiles256 <= device_sm_count() && K / PF_BK >= 8) {
    a.split = 1;
    return prefill_launch<256>(xq, B, a, N, pdl, st);
  }
  // otherwise 256-token tiles unless they would fill fewer than 3/4 of the SMs: then 128-token tiles
  if (tiles256 * 4 < static_cast<int64_t>(device_sm_count()) * 3) return prefill_launch<128>(xq, B, a, N, pdl, st);
  return prefill_launch<256>(xq, B, a, N, pdl, st);
}

}  // namespace paro
