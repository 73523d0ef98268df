// gemv1_b1.cu -- the one-token, one-launch decode kernel (B = 1): scale + L Givens layers +
// group-wise INT4 dequant GEMV in one launch per (multi-)linear.  This is the round-1 K-split
// kernel (16 compute warps + 1 producer warp in 96 registers, cp.async.bulk ring, IMMA tiles,
// cluster DSMEM reduction), kept as the single-launch B = 1 path because it measured faster than
// the generalised persistent-chain kernel of gemv1.cu for single launches (LLaMA-3-8B layer as
// four PDL launches: 34.3 vs 37.5 us, same box, tools/ab_step.py).  gemv1.cu runs chains and
// B > 1.  SURVEY.md 8(a) rows a4, a5, a6, a8.
//
// Work split: a cluster of CL CTAs owns a run of 32-row blocks of one linear; CTA c of the cluster
// owns the groups [c G / CL, (c + 1) G / CL) of those rows, transforms only its own groups (a warp
// per group) and streams only the tiles of its groups; the cluster sums its CTAs' row partials
// through DSMEM (st.async, fixed order) and the owner CTA of a row writes y.  Dot product on the
// warp-level integer tensor cores: x' as per-(group, token) 16-bit fixed point split in two s8
// digits, the u8 codes of an AND-masked code word as the A fragment, exact int32 per (row, group).
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "paro_internal.h"
#include "ptx.cuh"
#include "tile_layout.cuh"

namespace paro {

#ifndef PARO_TIMELINE
#define PARO_TIMELINE 0
#endif
#ifndef PARO_B1_KS_MIN_BYTES
#define PARO_B1_KS_MIN_BYTES 64e6  // weight stream from which a single long-K launch splits K over clusters
#endif
#ifndef PARO_B1_SHORT_MULTI_CAP
#define PARO_B1_SHORT_MULTI_CAP 1
#endif
#if PARO_TIMELINE
// per (CTA, launch slot, event) clock64 marks (tools/timeline_b1.py); launch slot = launch
// sequence number mod 16 (paro_debug_b1_seq_reset restarts it); event 11 = %globaltimer at event 0
__device__ unsigned long long g_tl_b1[1024 * 16 * 12];
static int g_b1_seq = 0;
extern "C" int paro_debug_timeline_b1(unsigned long long* host, int n) {
  if (n > 1024 * 16 * 12) n = 1024 * 16 * 12;
  return static_cast<int>(cudaMemcpyFromSymbol(host, g_tl_b1, sizeof(unsigned long long) * n));
}
extern "C" void paro_debug_b1_seq_reset() { g_b1_seq = 0; }
// per-stage marks of launch slots 12..15: [slot - 12][CTA][stage][0 producer issued, 1 consumer data-ready, 2 consumer done]
__device__ unsigned long long g_tl_b1_st[4 * 1024 * 64 * 3];
extern "C" int paro_debug_timeline_b1_st(unsigned long long* host, int n) {
  if (n > 4 * 1024 * 64 * 3) n = 4 * 1024 * 64 * 3;
  return static_cast<int>(cudaMemcpyFromSymbol(host, g_tl_b1_st, sizeof(unsigned long long) * n));
}
#endif
__device__ __forceinline__ void b1_mark(int slot, int ev) {
#if PARO_TIMELINE
  if (blockIdx.x < 1024) {
    unsigned long long c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
    g_tl_b1[(blockIdx.x * 16 + slot) * 12 + ev] = c;
    if (ev == 0) g_tl_b1[(blockIdx.x * 16 + slot) * 12 + 11] = globaltimer_ns();
  }
#else
  (void)slot;
  (void)ev;
#endif
}
#if PARO_TIMELINE
// per-tile marks of launch slot 13 (the step's o_proj): [CTA][warp][k-th tile of the warp]
__device__ unsigned long long g_tl_b1_tile[1024 * 16 * 4];
extern "C" int paro_debug_timeline_b1_tile(unsigned long long* host, int n) {
  if (n > 1024 * 16 * 4) n = 1024 * 16 * 4;
  return static_cast<int>(cudaMemcpyFromSymbol(host, g_tl_b1_tile, sizeof(unsigned long long) * n));
}
#endif
__device__ __forceinline__ void b1_mark_tile(int slot, int warp, int k) {
#if PARO_TIMELINE
  if (slot == 13 && blockIdx.x < 1024 && k < 4) {
    unsigned long long c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
    g_tl_b1_tile[(blockIdx.x * 16 + warp) * 4 + k] = c;
  }
#else
  (void)slot;
  (void)warp;
  (void)k;
#endif
}
__device__ __forceinline__ void b1_mark_st(int slot, int st, int ev) {
#if PARO_TIMELINE
  if (slot >= 12 && blockIdx.x < 1024 && st < 64) {
    unsigned long long c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
    g_tl_b1_st[(((slot - 12) * 1024 + blockIdx.x) * 64 + st) * 3 + ev] = c;
  }
#else
  (void)slot;
  (void)st;
  (void)ev;
#endif
}

namespace {
constexpr int B1_NW = 16;  // compute warps per CTA (+ 1 producer warp)
constexpr uint32_t TILE_B = TILE_CODE_BYTES + TILE_SCALE_BYTES + TILE_ZERO_BYTES;

// D(16x8 s32) += A(16x32 u8, row) * B(32x8 s8, col); fragments as in ptx.cuh (imma_16832),
// not volatile so the scheduler may interleave the four accumulator chains
__device__ __forceinline__ void mma_u8s8(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
  asm("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

}  // namespace

// NW compute warps + 1 producer warp (17 warps: up to 96 registers per thread).
// BT: token capacity of the instance (1, 4, 8, 16).  Tokens are transformed four at a time in
// lockstep and occupy the MMA's 8 columns in sets of four (columns 2b, 2b+1 = hi, lo digit of
// token b of the set).  BT = 1 sums row partials per warp in a fixed order (deterministic);
// BT > 1 adds them with shared-memory atomics.
// MODE: 0 the regular epilogue, 1 the cross-cluster K split (a.KS > 1), 2 the NVLink peer-store
// all-gather (a.p2p) -- each its own instance, so the regular one carries none of the others' code.
// ATM: row partials added with shared-memory atomics (a.atom; many rows per cluster)
template <int NW, int BT, int MODE, bool ATM>
__global__ void __launch_bounds__((NW + 1) * 32, 1) paro_gemv1_b1_kernel(const B1Args a) {
  constexpr int TB = BT == 1 ? 1 : 4;          // tokens per transform chunk / MMA column set
  constexpr int NB = (BT + 3) / 4;             // column sets
  constexpr int NCOL = BT == 1 ? 2 : 8;        // B columns holding digits
  constexpr int XTQ = NCOL * 32;               // digit bytes per (group, set, quad)
  constexpr int XPC = 4 * XTQ;                 // digit bytes per (group, column set)
  constexpr int XPG = NB * XPC;                // digit bytes per group
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int li = 0;
#pragma unroll 1
  while (li + 1 < a.n_lin && static_cast<int>(blockIdx.x) >= a.lin[li + 1].cta_begin) ++li;
  const B1Linear& d = a.lin[li];
  const int CL = static_cast<int>(cluster_nctarank());
  const int crank = static_cast<int>(cluster_ctarank());
  const int G = a.G, B = a.B;
  const int KS = MODE == 1 ? a.KS : 1;
  const int cl_all = (static_cast<int>(blockIdx.x) - d.cta_begin) / CL;
  const int kq = cl_all % KS, cl = cl_all / KS;  // K slice, row range
  const int nrb = d.rb_base + (cl < d.rb_extra ? 1 : 0);
  const int rb0 = cl * d.rb_base + min(cl, d.rb_extra);
  const int R = nrb * TILE_ROWS;
  const int gs0 = kq * G / KS, Gs = (kq + 1) * G / KS - gs0;
  const int ga = gs0 + crank * Gs / CL, gb = gs0 + (crank + 1) * Gs / CL, gc = gb - ga;
  // stages: TPS consecutive tiles of the CTA's tile sequence u = rb * gc + (gamma - ga)
  // (row block by row block, my groups within each; a stage may start or end inside a row block)
  const int n_tiles = nrb * gc;
  const int n_stages = (n_tiles + a.TPS - 1) / a.TPS;

  uint8_t* xp = smem + a.off_xp;                                 // x' digits [gc][NB][4 t][NCOL][4 kb][8 B]
  int2* xs = reinterpret_cast<int2*>(smem + a.off_xs);           // per (group, token): (sum x'fix, 2^(E-14))
  const uint8_t* zblk = smem + a.off_xs + ((gc * BT * 8 + 15) & ~15);  // 32 zero bytes (B columns >= 2)
  float* part = reinterpret_cast<float*>(smem + a.off_part);     // BT = 1: [NW][R_max]; else [R_max][BT]
  float* recv = reinterpret_cast<float*>(smem + a.off_recv);     // [CL][RRmax][BT] cluster partials
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.off_bar);
  uint64_t* empty = full + a.S;
  uint64_t* rbar = empty + a.S;  // cluster partials of my rows landed (st.async bytes)
  uint64_t* xbar = rbar + 1;     // BT > 1: the pre-transformed x' slice landed
  const int RR = (R + CL - 1) / CL;  // rows per owner CTA
  const int my_lo = crank * RR, my_n = max(0, min(RR, R - my_lo));
  uint8_t* ring = smem + a.off_ring;

  if (threadIdx.x < 8) reinterpret_cast<uint32_t*>(smem + a.off_xs + ((gc * BT * 8 + 15) & ~15))[threadIdx.x] = 0u;
  if (threadIdx.x == 0) {
    for (int i = 0; i < a.S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NW);
    }
    mbar_init(rbar, 1);
    mbar_init(xbar, 1);
    if (CL > 1) mbar_arrive_expect_tx(rbar, static_cast<uint32_t>((CL - 1) * my_n * BT * 4));
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) b1_mark(a.tl_slot, 0);
  // BT > 1: the cluster barrier arrive of the compute warps comes after phase 1, because the
  // transform scratch shares its shared memory with recv, which other CTAs write once the
  // barrier completes
  if (CL > 1 && (BT == 1 || warp == NW)) cluster_arrive_relaxed();
  if (a.pdl) pdl_launch_dependents();

  // ------------------------------------------------------------ producer warp: the whole ring
  if (warp == NW) {
    const uint64_t pol = l2_evict_first_policy();
    const int pre = min(a.pre_stages, n_stages);
    auto issue_xq = [&]() {  // BT > 1: x' digits of my groups, written by the preceding xform kernel
      if (a.pdl) pdl_wait();
      if (lane == 0) {
        const uint32_t nd = static_cast<uint32_t>(gc * XPG), ns = static_cast<uint32_t>(gc * BT * 8);
        mbar_arrive_expect_tx(xbar, nd + ns);
        bulk_g2s_nohint(xp, d.xq + static_cast<size_t>(ga) * XPG, nd, xbar);
        bulk_g2s_nohint(xs, d.xqs + static_cast<size_t>(ga) * BT, ns, xbar);
      }
      __syncwarp();
    };
    if (a.params_first) named_bar_sync(3, (NW + 1) * 32);  // the rotation-parameter loads are out
    if (lane == 0) b1_mark(a.tl_slot, 10);
#pragma unroll 1
    for (int st = 0; st < n_stages; ++st) {
      const int slot = st % a.S;
      // the latency-critical x / rotation-parameter loads of the compute warps go out before
      // the bulk of the weight stream (which would otherwise queue ahead of them)
      if (st == pre) {
        if (BT > 1) issue_xq();
        named_bar_sync(2, (NW + 1) * 32);
        if (lane == 0) b1_mark(a.tl_slot, 9);
      }
      if (st >= a.S) mbar_wait(&empty[slot], ((st / a.S) & 1) ^ 1);
      if (lane == 0) {
        const int u0 = st * a.TPS, u1 = min(n_tiles, u0 + a.TPS);
        uint8_t* dst = ring + static_cast<size_t>(slot) * a.slot_bytes;
        mbar_arrive_expect_tx(&full[slot], static_cast<uint32_t>(u1 - u0) * TILE_B);
#pragma unroll 1
        for (int u = u0; u < u1;) {  // one contiguous segment per row block touched
          const int rb = u / gc, ue = min(u1, (rb + 1) * gc);
          const int64_t T = static_cast<int64_t>(rb0 + rb) * G + ga + (u - rb * gc);
          const uint32_t i0 = static_cast<uint32_t>(u - u0), n = static_cast<uint32_t>(ue - u);
          u = ue;
          bulk_g2s(dst + i0 * TILE_CODE_BYTES, d.codes + T * TILE_CODE_BYTES, n * TILE_CODE_BYTES, &full[slot], pol);
          bulk_g2s(dst + a.sc_off + i0 * TILE_SCALE_BYTES, d.scales + T * TILE_SCALE_BYTES, n * TILE_SCALE_BYTES,
                   &full[slot], pol);
          bulk_g2s(dst + a.z_off + i0 * TILE_ZERO_BYTES, d.zeros + T * TILE_ZERO_BYTES, n * TILE_ZERO_BYTES, &full[slot],
                   pol);
        }
        b1_mark_st(a.tl_slot, st, 0);
      }
      __syncwarp();
    }
    if (lane == 0) b1_mark(a.tl_slot, 8);
    if (pre >= n_stages) {
      if (BT > 1) issue_xq();
      named_bar_sync(2, (NW + 1) * 32);
    }
    if (CL > 1) cluster_wait();
    return;
  }

  // ------------------------------------------------------------ phase 1: x' of my groups (a4, a5)
  float* pw = part + static_cast<size_t>(warp) * a.R_max;
  if (BT == 1 && !ATM) {
    for (int i = lane; i < R; i += 32) pw[i] = 0.f;
  } else {
    for (int i = threadIdx.x; i < R * BT; i += NW * 32) part[i] = 0.f;
  }
  if constexpr (BT > 1) {
    // x' digits and (sum, scale) of my groups come from paro_gemv1_xform_kernel (one transform
    // per (group, token) for the whole GPU instead of one per cluster): the producer bulk-copies
    // the contiguous slice [ga, gb) after the PDL wait
    if (a.params_first) named_bar_arrive(3, (NW + 1) * 32);
    named_bar_arrive(2, (NW + 1) * 32);
    if (a.pdl) pdl_wait();  // (y is written at the end)
    mbar_wait(xbar, 0);
  } else {
    float* scr = reinterpret_cast<float*>(smem + a.off_scr) + warp * (TB * 128);
    const int L = a.rotate ? d.L : 0;
    bool waited = false, arrived = false;
    if (warp >= gc) {
      if (a.params_first) named_bar_arrive(3, (NW + 1) * 32);
      named_bar_arrive(2, (NW + 1) * 32);
    } else if (lane == 0) {
      // later rounds' rotation records -> L2 now, ahead of the weight stream (requested after
      // the first round they would queue behind the whole ring)
      for (int g = warp + NW; g < gc; g += NW) {
        const int64_t rec = static_cast<int64_t>(ga + g) * L * 32;
        if (L > 0) {
          prefetch_l2_bulk(reinterpret_cast<const float4*>(d.rot_cs) + rec, static_cast<uint32_t>(L * 32 * 16));
          prefetch_l2_bulk(reinterpret_cast<const uint32_t*>(d.rot_idx) + rec, static_cast<uint32_t>(L * 32 * 4));
        }
        if (a.rotate) prefetch_l2_bulk(d.svec + (ga + g) * 128, 512u);
      }
    }
#pragma unroll 1
    for (int g = warp; g < gc; g += NW) {
      const int gam = ga + g;
      // rotation records [group][layer][32 lanes]: (cos, sin) of slots lane, lane + 32 and
      // their (i, j) channel pairs (pack-time bank-conflict-free schedule)
      float4 cs[8];
      uint32_t ix[8];
      const int64_t rec = static_cast<int64_t>(gam) * L * 32 + lane;
#pragma unroll
      for (int t = 0; t < 8; ++t)
        if (t < L) {
          cs[t] = __ldg(reinterpret_cast<const float4*>(d.rot_cs) + rec + t * 32);
          ix[t] = __ldg(reinterpret_cast<const uint32_t*>(d.rot_idx) + rec + t * 32);
        }
      const float4 sv =
          a.rotate ? __ldg(reinterpret_cast<const float4*>(d.svec + gam * 128) + lane) : make_float4(1.f, 1.f, 1.f, 1.f);
      if (!waited && a.params_first) {
        __syncwarp();
        named_bar_arrive(3, (NW + 1) * 32);
      }
      if (!waited) {
        if (a.pdl) pdl_wait();  // x may be written by the previous kernel on the stream
        waited = true;
        if (warp == 0 && lane == 0) b1_mark(a.tl_slot, 1);
      }
#pragma unroll 1
      for (int b0 = 0; b0 < B; b0 += TB) {  // token chunks, TB tokens in lockstep
        uint2 xv[TB];
#pragma unroll
        for (int tb = 0; tb < TB; ++tb)
          xv[tb] = (b0 + tb < B) ? __ldg(reinterpret_cast<const uint2*>(static_cast<const uint8_t*>(a.x) +
                                                                       (static_cast<int64_t>(b0 + tb) * a.K +
                                                                        gam * 128 + 4 * lane) * 2))
                                 : make_uint2(0u, 0u);  // tokens >= B: x = 0, never stored
#pragma unroll
        for (int tb = 0; tb < TB; ++tb) {
          float2 f01, f23;
          if (a.x_bf16) {
            f01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xv[tb].x));
            f23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xv[tb].y));
          } else {
            f01 = __half22float2(*reinterpret_cast<const __half2*>(&xv[tb].x));
            f23 = __half22float2(*reinterpret_cast<const __half2*>(&xv[tb].y));
          }
          // a4: u = s . x
          *reinterpret_cast<float4*>(scr + tb * 128 + 4 * lane) =
              make_float4(f01.x * sv.x, f01.y * sv.y, f23.x * sv.z, f23.y * sv.w);
        }
        if (!arrived) {
          __syncwarp();
          named_bar_arrive(2, (NW + 1) * 32);  // my x and parameters are in
          arrived = true;
          if (warp == 0 && lane == 0) b1_mark(a.tl_slot, 2);
        }
        __syncwarp();
        // a5: rotations t = 1..L, each pair from the pre-update values (Eq. 4 / Eq. 5)
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          if (t >= L) break;
          const uint32_t i0 = ix[t] & 0xff, j0 = (ix[t] >> 8) & 0xff, i1 = (ix[t] >> 16) & 0xff, j1 = ix[t] >> 24;
#pragma unroll
          for (int tb = 0; tb < TB; ++tb) {
            float* sc = scr + tb * 128;
            const float a0 = sc[i0], b0v = sc[j0], a1 = sc[i1], b1v = sc[j1];
            sc[i0] = cs[t].x * a0 - cs[t].y * b0v;
            sc[j0] = cs[t].y * a0 + cs[t].x * b0v;
            sc[i1] = cs[t].z * a1 - cs[t].w * b1v;
            sc[j1] = cs[t].w * a1 + cs[t].z * b1v;
          }
          __syncwarp();
        }
        // x' -> per-(group, token) fixed point and s8 digits (see the header), laid out as B
        // fragments [column set][quad t][column][k-block kb][b0, b1]; column 2 b + dg of a set =
        // digit dg (0 hi, 1 lo) of its token b; k-block kb = 2 p + h covers the low (p = 0) or
        // high (p = 1) nibbles of words 2h, 2h + 1 (b0: word 2h, b1: word 2h + 1); byte bb of the
        // word for quad t, word j, parity p is channel tile_k(t, j, 2 bb + p)
#pragma unroll
        for (int tb = 0; tb < TB; ++tb) {
          int* fx = reinterpret_cast<int*>(scr + tb * 128);
          const float4 v = *reinterpret_cast<const float4*>(scr + tb * 128 + 4 * lane);
          const float ml = fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w)));
          const uint32_t mb = __reduce_max_sync(0xffffffffu, __float_as_uint(ml));  // |x| bits order like |x|
          int E = mb < 0x00800000u ? -100 : static_cast<int>(mb >> 23) - 127 + ((mb & 0x7fffffu) != 0u ? 1 : 0);
          E = max(E, -100);
          const float mul = __uint_as_float(static_cast<uint32_t>(141 - E) << 23);  // 2^(14 - E)
          const int f0 = __float2int_rn(v.x * mul), f1 = __float2int_rn(v.y * mul);
          const int f2 = __float2int_rn(v.z * mul), f3 = __float2int_rn(v.w * mul);
          const int X = __reduce_add_sync(0xffffffffu, (f0 + f1) + (f2 + f3));
          __syncwarp();  // every lane has read its x' before the scratch holds x'fix
          *reinterpret_cast<int4*>(fx + 4 * lane) = make_int4(f0, f1, f2, f3);
          __syncwarp();
          const int tq = lane >> 3, col = (lane >> 2) & 1, kb = lane & 3, p = kb >> 1, h = kb & 1;
          uint32_t wd[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int j = 2 * h + e;
            uint32_t wv = 0;
#pragma unroll
            for (int bb = 0; bb < 4; ++bb) {
              const int c = 16 * (2 * j + p) + 2 * tq + (bb >> 1) + 8 * (bb & 1);  // tile_k(tq, j, 2 bb + p)
              const int f = fx[c];
              const int lo = static_cast<int>(static_cast<int8_t>(f & 0xff));
              const int dg = col ? lo : ((f - lo) >> 8);
              wv |= (static_cast<uint32_t>(dg) & 0xffu) << (8 * bb);
            }
            wd[e] = wv;
          }
          const int b = b0 + tb, set = b >> 2, cb = b & 3;
          *reinterpret_cast<uint2*>(xp + g * XPG + set * XPC + tq * XTQ + (2 * cb + col) * 32 + kb * 8) =
              make_uint2(wd[0], wd[1]);
          if (lane == 0)
            xs[g * BT + b] = make_int2(X, static_cast<int>(static_cast<uint32_t>(113 + E) << 23));  // 2^(E - 14)
        }
        __syncwarp();
      }
    }
  }
  named_bar_sync(1, NW * 32);  // every x' of the CTA is in shared memory (and BT > 1: part zeroed)
  if (threadIdx.x == 0) b1_mark(a.tl_slot, 3);
  if (BT > 1 && CL > 1) cluster_arrive();  // my scratch is free: the cluster may now write recv

  // ------------------------------------------------------------ phase 2: tiles (a6)
  {
    const int gq = lane >> 2, tq = lane & 3;
    constexpr bool atom = ATM;
    // stage bookkeeping advanced incrementally (no divisions in the loop): ring slot and phase,
    // first tile u0 = st * TPS = r_lo * gc + off0
    int slot = 0, phase = 0, r_lo = 0, off0 = 0;
    for (int st = 0; st < n_stages; ++st) {
      // stage tiles [u0, u1): tile i of the stage is (row block r_lo + ri, group ga + gi) with
      // (ri, gi) = divmod(off0 + i, gc)
      const int u0 = st * a.TPS, nt = min(n_tiles, u0 + a.TPS) - u0;
      const int g_lo = ga, pl = gc;
      mbar_wait(&full[slot], phase);
      if (st == 0 && threadIdx.x == 0) b1_mark(a.tl_slot, 4);
      if (threadIdx.x == 0) b1_mark_st(a.tl_slot, st, 1);
      const uint8_t* sb = ring + static_cast<size_t>(slot) * a.slot_bytes;
      if constexpr (BT == 1) {
      int ri = 0, gi = off0 + warp;  // tile warp + k NW of the stage
      while (gi >= pl) {
        gi -= pl;
        ++ri;
      }
#pragma unroll 1
      for (int i = warp; i < nt; i += NW) {
        const int gl = g_lo - ga + gi;
        const uint8_t* tc = sb + i * TILE_CODE_BYTES + gq * 64 + tq * 16;
        uint4 w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) w[q] = *reinterpret_cast<const uint4*>(tc + q * 512);
        const uint2 sp = *reinterpret_cast<const uint2*>(sb + a.sc_off + i * TILE_SCALE_BYTES + gq * 8);
        const uint32_t zw = *reinterpret_cast<const uint16_t*>(sb + a.z_off + i * TILE_ZERO_BYTES + gq * 2);
        const float2 Sa = __half22float2(*reinterpret_cast<const __half2*>(&sp.x));  // rows gq, gq + 8
        const float2 Sb = __half22float2(*reinterpret_cast<const __half2*>(&sp.y));  // rows gq + 16, gq + 24
        const float Sr[4] = {Sa.x, Sa.y, Sb.x, Sb.y};
        const int rowl = (r_lo + ri) * TILE_ROWS + gq;  // cluster-local row of q = 0
#pragma unroll
        for (int set = 0; set < NB; ++set) {
          if (set * 4 >= B) break;
          // B fragments: lanes of MMA columns >= 2 read a 32-byte zero block (address select, no branch)
          const uint8_t* bp = gq < 2 ? xp + gl * XPG + set * XPC + tq * XTQ + gq * 32 : zblk;
          const uint4 bA = *reinterpret_cast<const uint4*>(bp);
          const uint4 bB = *reinterpret_cast<const uint4*>(bp + 16);
          constexpr uint32_t ML = 0x0f0f0f0fu, MH = 0xf0f0f0f0u;
          int Dl[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}}, Dh[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {  // rows gq + 16 hh (w[2 hh]) and gq + 16 hh + 8 (w[2 hh + 1])
            const uint4 r0 = w[2 * hh], r1 = w[2 * hh + 1];
            mma_u8s8(Dl[hh], r0.x & ML, r1.x & ML, r0.y & ML, r1.y & ML, bA.x, bA.y);  // low nibbles, words 0, 1
            mma_u8s8(Dl[hh], r0.z & ML, r1.z & ML, r0.w & ML, r1.w & ML, bA.z, bA.w);  // low nibbles, words 2, 3
            mma_u8s8(Dh[hh], r0.x & MH, r1.x & MH, r0.y & MH, r1.y & MH, bB.x, bB.y);  // high nibbles (16 q)
            mma_u8s8(Dh[hh], r0.z & MH, r1.z & MH, r0.w & MH, r1.w & MH, bB.z, bB.w);
          }
          // lane (gq, tq) holds columns 2 tq (hi digit) and 2 tq + 1 (lo digit) = token tq of the
          // set, rows gq + 8 q
          const int b = set * 4 + tq;
          if (BT == 1 ? tq == 0 : b < B) {
            const int2 xf = xs[gl * BT + b];
            const float F = __int_as_float(xf.y);
            float out[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int hh = q >> 1, e = (q & 1) * 2;
              const int zq = static_cast<int>((zw >> (4 * q)) & 15u);
              const int I = Dl[hh][e] * 256 + Dl[hh][e + 1] + ((Dh[hh][e] * 256 + Dh[hh][e + 1]) >> 4) - zq * xf.x;
              out[q] = Sr[q] * F * static_cast<float>(I);
            }
            if (BT == 1 && !atom) {  // one uniform branch per tile, not per row
#pragma unroll
              for (int q = 0; q < 4; ++q) pw[rowl + 8 * q] += out[q];
            } else {
#pragma unroll
              for (int q = 0; q < 4; ++q) atomicAdd(part + (rowl + 8 * q) * BT + b, out[q]);
            }
          }
        }
        if (lane == 0 && st == 0) b1_mark_tile(a.tl_slot, warp, (i - warp) / NW);
        gi += NW;
        while (gi >= pl) {
          gi -= pl;
          ++ri;
        }
      }
      } else {
      // B > 1: warp w takes a contiguous chunk of the stage's tiles (row block ri, group gi), so
      // that its consecutive tiles mostly share a row block and the row partials (atomics) go to
      // shared memory once per row block; B = 1: tiles w, w + NW, ... (measured faster)
      const int per = (nt + NW - 1) / NW;
      const int step = BT == 1 ? NW : 1;
      const int i_end = BT == 1 ? nt : min(nt, (warp + 1) * per);
      int i = BT == 1 ? warp : warp * per;
      int ri = (off0 + i) / pl, gi = off0 + i - ri * pl;
      float acc[NB][4];
      int acc_ri = -1;
      auto flush = [&]() {
        if (acc_ri < 0) return;
        const int rowl = (r_lo + acc_ri) * TILE_ROWS + gq;  // cluster-local row of q = 0
#pragma unroll
        for (int set = 0; set < NB; ++set) {
          const int b = set * 4 + tq;
          if (BT == 1 ? tq == 0 : b < B) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              if (BT == 1)
                pw[rowl + 8 * q] += acc[set][q];
              else
                atomicAdd(part + (rowl + 8 * q) * BT + b, acc[set][q]);
            }
          }
        }
      };
#pragma unroll 1
      for (; i < i_end; i += step) {
        if (ri != acc_ri) {
          flush();
          acc_ri = ri;
#pragma unroll
          for (int set = 0; set < NB; ++set)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[set][q] = 0.f;
        }
        const int gl = g_lo - ga + gi;
        const uint8_t* tc = sb + i * TILE_CODE_BYTES + gq * 64 + tq * 16;
        uint4 w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) w[q] = *reinterpret_cast<const uint4*>(tc + q * 512);
        const uint2 sp = *reinterpret_cast<const uint2*>(sb + a.sc_off + i * TILE_SCALE_BYTES + gq * 8);
        const uint32_t zw = *reinterpret_cast<const uint16_t*>(sb + a.z_off + i * TILE_ZERO_BYTES + gq * 2);
        const float2 Sa = __half22float2(*reinterpret_cast<const __half2*>(&sp.x));  // rows gq, gq + 8
        const float2 Sb = __half22float2(*reinterpret_cast<const __half2*>(&sp.y));  // rows gq + 16, gq + 24
        const float Sr[4] = {Sa.x, Sa.y, Sb.x, Sb.y};
#pragma unroll
        for (int set = 0; set < NB; ++set) {
          if (set * 4 >= B) break;
          uint4 bA = make_uint4(0u, 0u, 0u, 0u), bB = bA;  // B fragments (columns >= NCOL are zero)
          if (gq < NCOL) {
            const uint8_t* bp = xp + gl * XPG + set * XPC + tq * XTQ + gq * 32;
            bA = *reinterpret_cast<const uint4*>(bp);
            bB = *reinterpret_cast<const uint4*>(bp + 16);
          }
          constexpr uint32_t ML = 0x0f0f0f0fu, MH = 0xf0f0f0f0u;
          int Dl[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}}, Dh[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {  // rows gq + 16 hh (w[2 hh]) and gq + 16 hh + 8 (w[2 hh + 1])
            const uint4 r0 = w[2 * hh], r1 = w[2 * hh + 1];
            mma_u8s8(Dl[hh], r0.x & ML, r1.x & ML, r0.y & ML, r1.y & ML, bA.x, bA.y);  // low nibbles, words 0, 1
            mma_u8s8(Dl[hh], r0.z & ML, r1.z & ML, r0.w & ML, r1.w & ML, bA.z, bA.w);  // low nibbles, words 2, 3
            mma_u8s8(Dh[hh], r0.x & MH, r1.x & MH, r0.y & MH, r1.y & MH, bB.x, bB.y);  // high nibbles (16 q)
            mma_u8s8(Dh[hh], r0.z & MH, r1.z & MH, r0.w & MH, r1.w & MH, bB.z, bB.w);
          }
          // lane (gq, tq) holds columns 2 tq (hi digit) and 2 tq + 1 (lo digit) = token tq of the
          // set, rows gq + 8 q
          const int b = set * 4 + tq;
          if (BT == 1 ? tq == 0 : b < B) {
            const int2 xf = xs[gl * BT + b];
            const float F = __int_as_float(xf.y);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int hh = q >> 1, e = (q & 1) * 2;
              const int zq = static_cast<int>((zw >> (4 * q)) & 15u);
              const int I = Dl[hh][e] * 256 + Dl[hh][e + 1] + ((Dh[hh][e] * 256 + Dh[hh][e + 1]) >> 4) - zq * xf.x;
              acc[set][q] = fmaf(Sr[q] * F, static_cast<float>(I), acc[set][q]);
            }
          }
        }
        gi += step;
        while (gi >= pl) {
          gi -= pl;
          ++ri;
        }
      }
      flush();
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      if (threadIdx.x == 0) b1_mark_st(a.tl_slot, st, 2);
      if (++slot == a.S) {
        slot = 0;
        phase ^= 1;
      }
      off0 += a.TPS;
      while (off0 >= gc) {
        off0 -= gc;
        ++r_lo;
      }
    }
  }

  // ------------------------------------------------------------ reduction + epilogue (a8)
  named_bar_sync(1, NW * 32);
  if (threadIdx.x == 0) b1_mark(a.tl_slot, 5);
  if (CL > 1) cluster_wait();  // every CTA of the cluster is running: DSMEM is legal
  const int tid = threadIdx.x;
  for (int idx = tid; idx < R * BT; idx += NW * 32) {
    const int r = idx / BT, b = idx - r * BT;
    float sum;
    if (BT == 1 && !ATM) {
      float s4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
      for (int w = 0; w < NW; ++w) s4[w & 3] += part[static_cast<size_t>(w) * a.R_max + r];
      sum = (s4[0] + s4[1]) + (s4[2] + s4[3]);  // fixed order
    } else {
      sum = part[idx];
    }
    const int owner = r / RR;
    float* dst = recv + (crank * a.RRmax + (r - owner * RR)) * BT + b;
    if (owner == crank)
      *dst = sum;
    else
      st_async_b32(mapa(smem_u32(dst), static_cast<uint32_t>(owner)), __float_as_uint(sum),
                   mapa(smem_u32(rbar), static_cast<uint32_t>(owner)));
  }
  named_bar_sync(1, NW * 32);  // my own partials are in recv
  if (CL > 1) mbar_wait(rbar, 0);  // and those of the other CTAs of the cluster
  if (threadIdx.x == 0) b1_mark(a.tl_slot, 6);
  if (a.pdl) pdl_wait();  // y may still be read by the previous kernel
  for (int idx = tid; idx < my_n * BT; idx += NW * 32) {
    const int rl = idx / BT, b = idx - rl * BT;
    if (b >= B) continue;
    float v = 0.f;
    for (int c = 0; c < CL; ++c) v += recv[(c * a.RRmax + rl) * BT + b];  // fixed order
    const int64_t n = static_cast<int64_t>(rb0) * TILE_ROWS + my_lo + rl;
    if (KS > 1) {  // my K slice's row sums: the last cluster of the row range adds them below
      if (n < d.N) __stcg(a.ks_part + static_cast<int64_t>(kq) * d.N + n, v);
      continue;
    }
    if (n < d.N) {
      if (d.bias) v += __ldg(d.bias + n);
      if (MODE != 2) {
        const int64_t o = static_cast<int64_t>(b) * d.N + n;
        if (a.y_dtype == 0)
          static_cast<__half*>(d.y)[o] = __float2half_rn(v);
        else if (a.y_dtype == 1)
          static_cast<__nv_bfloat16*>(d.y)[o] = __float2bfloat16_rn(v);
        else
          static_cast<float*>(d.y)[o] = v;
      } else {
        // NVLink-native all-gather: this rank's columns of every rank's y_full (P2P stores)
        const int64_t o = static_cast<int64_t>(b) * a.y_ld + a.y_col0 + n;
        for (int p = 0; p < a.world; ++p) {
          if (a.y_dtype == 0)
            static_cast<__half*>(a.peer_y[p])[o] = __float2half_rn(v);
          else if (a.y_dtype == 1)
            static_cast<__nv_bfloat16*>(a.peer_y[p])[o] = __float2bfloat16_rn(v);
          else
            static_cast<float*>(a.peer_y[p])[o] = v;
        }
      }
    }
  }
  if (KS > 1) {
    // last-arriver reduction over the KS clusters of this row range (no waiting: the CTA that
    // completes the count adds the slices in the fixed order 0..KS-1 and stores y)
    volatile int& s_last = *reinterpret_cast<int*>(smem + a.off_xs);  // x' sums are no longer read
    __threadfence();  // my row sums are visible at GPU scope before the count below
    named_bar_sync(1, NW * 32);
    if (tid == 0) {
      uint32_t* ctr = a.ks_ctr + (d.cta_begin / (CL * KS) + cl) * CL + crank;
      const uint32_t old = atomicAdd(ctr, 1u);
      const int last = old == static_cast<uint32_t>(KS - 1);
      if (last) {
        *ctr = 0u;  // every CTA of this row range has counted: ready for the next call
        __threadfence();
      }
      s_last = last;
    }
    named_bar_sync(1, NW * 32);
    if (s_last) {
      for (int rl = tid; rl < my_n; rl += NW * 32) {
        const int64_t n = static_cast<int64_t>(rb0) * TILE_ROWS + my_lo + rl;
        if (n >= d.N) continue;
        float v = 0.f;
        for (int q = 0; q < KS; ++q) v += __ldcg(a.ks_part + static_cast<int64_t>(q) * d.N + n);  // fixed order
        if (d.bias) v += __ldg(d.bias + n);
        if (a.y_dtype == 0)
          static_cast<__half*>(d.y)[n] = __float2half_rn(v);
        else if (a.y_dtype == 1)
          static_cast<__nv_bfloat16*>(d.y)[n] = __float2bfloat16_rn(v);
        else
          static_cast<float*>(d.y)[n] = v;
      }
    }
  }
  if (threadIdx.x == 0) b1_mark(a.tl_slot, 7);
  if (MODE == 2) {
    // every CTA's peer stores are ordered before its arrival (release at GPU scope); the last CTA to
    // arrive acquires them all and its system-scope release -- cumulative over what it observed --
    // publishes this rank's flag on every rank
    named_bar_sync(1, NW * 32);
    if (tid == 0) {
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      uint32_t old;
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(a.done_ctr) : "memory");
      if (old == gridDim.x - 1) {
        asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(a.done_ctr) : "memory");
        asm volatile("fence.acq_rel.sys;" ::: "memory");
        const uint32_t e = *a.epoch + 1u;
        for (int p = 0; p < a.world; ++p)
          asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a.peer_flags[p] + a.rank), "r"(e) : "memory");
      }
    }
  }
}

// The consumer side of the NVLink-native all-gather: one thread waits until every rank released
// its flag for this exchange (epoch + 1), then advances the local epoch.
__global__ void p2p_wait_kernel(uint32_t* flags, uint32_t* epoch, int world) {
  // the next kernel may start its prologue (weight prefetch) now; its PDL wait still waits for this
  // kernel's completion before it reads y_full
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x != 0) return;
  const uint32_t e = *epoch + 1u;
  const uint64_t t0 = globaltimer_ns();
  for (int q = 0; q < world; ++q) {
    for (;;) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + q) : "memory");
      if (static_cast<int>(v - e) >= 0) break;
      if (globaltimer_ns() - t0 > 4000000000ull) __trap();  // a peer never signalled
    }
  }
  *epoch = e;
}

cudaError_t launch_p2p_wait(uint32_t* flags, uint32_t* epoch, int world, int pdl, cudaStream_t st) {
  // under PDL the wait starts while the GEMV still runs (the GEMV triggers its dependents at its
  // start): it only polls flags the GEMV's last CTA releases, and reads the epoch, which the
  // previous wait kernel wrote before this GEMV could start
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(32);
  cfg.stream = st;
  cudaLaunchAttribute at;
  at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at.val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = &at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, p2p_wait_kernel, flags, epoch, world);
}


// ============================================================================ host side
static int b1_env(const char* name, int dflt) {
#if PARO_DEBUG_KNOBS
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
#else
  (void)name;
  return dflt;
#endif
}

static inline uint32_t b1_align(uint32_t v, uint32_t al) { return (v + al - 1) / al * al; }

// clusters of CL (BT-token instance) that fit in one wave, from the occupancy API (cached per
// device)
static int b1_active_clusters_compute(const void* k, int CL, int threads, int budget) {
  ensure_smem_attr(k, budget);
  if (CL > 1) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(CL * 64);
  lc.blockDim = dim3(threads);
  lc.dynamicSmemBytes = budget;
  cudaLaunchAttribute at;
  at.id = cudaLaunchAttributeClusterDimension;
  at.val.clusterDim.x = CL;
  at.val.clusterDim.y = 1;
  at.val.clusterDim.z = 1;
  lc.attrs = &at;
  lc.numAttrs = 1;
  int nc = 0;
  if (cudaOccupancyMaxActiveClusters(&nc, k, &lc) != cudaSuccess || nc <= 0) {
    cudaGetLastError();
    nc = device_sm_count() / CL;
  }
  return nc;
}
static int b1_active_clusters(int BT, int CL, int threads, int budget) {
  (void)BT;
  return cached_device_int(reinterpret_cast<const void*>(&paro_gemv1_b1_kernel<B1_NW, 1, 0, false>), CL, threads, budget,
                           b1_active_clusters_compute);
}

// Cluster size = how many ways a row block's groups are split (G / CL groups transformed per CTA).
// The rotations are shared-memory bound (8 accesses per pair-update, all warps at once), so fewer
// groups per CTA shorten the transform; but clusters of 2 / 4 / 8 fill only 148 / 132 / 120 SMs
// (occupancy API), which slows the weight stream.  Measured (tools/time_groups.py,
// tools/time_70b.py): short streams (< 20 MB) at K = 4096 prefer 4, long ones 2; K >= 8192 prefers 8
// (one transform round) unless the stream is very long and G small (70B gate+up: 2).
static int b1_cluster_size(int n_lin, const int64_t* Ns, int64_t K, double* wbytes_out) {
  const int G = static_cast<int>(K / 128);
  double wbytes = 0;
  for (int i = 0; i < n_lin; ++i) wbytes += static_cast<double>(Ns[i]) * K * 0.52;
  int CL;
  if (G >= 64)
    CL = (wbytes < 64e6 || G >= 128) ? 8 : 2;
  else
    CL = wbytes < 20e6 ? 4 : 2;
  CL = b1_env("PARO_G1_CL", CL);
  if (G >= 64) CL = b1_env("PARO_G1_CL_BIGK", CL);
  if (CL < 1 || CL > 8) CL = 2;
  while (CL > 1 && CL > G) CL /= 2;
  if (wbytes_out) *wbytes_out = wbytes;
  return CL;
}

// Cross-cluster K split: a single long-K linear whose stream is long (>= 64 MB: LLaMA-3-70B
// down_proj) runs on clusters of 2 (148 SMs) instead of 8 (120 SMs), its K range split over KS
// clusters so that every CTA still transforms at most 16 groups (one round).  Shorter streams
// (LLaMA-3-8B / Qwen3-4B down_proj) measured slower with the split: the global last-arriver
// reduction costs more than the extra SMs bring (tools/ab_flag.sh).
int b1_ks_slices(int n_lin, const int64_t* Ns, int64_t K) {
  double wbytes = 0;
  const int CL = b1_cluster_size(n_lin, Ns, K, &wbytes);
  if (n_lin != 1 || CL != 8 || wbytes < PARO_B1_KS_MIN_BYTES) return 1;
  const int G = static_cast<int>(K / 128);
  const int ks = (G + 2 * B1_NW - 1) / (2 * B1_NW);
  return ks > 1 ? ks : 1;
}

size_t b1_ks_bytes(int KS, int64_t N) {
  return KS > 1 ? (static_cast<size_t>(KS * N * 4) + 255) / 256 * 256 : 0;
}

bool plan_gemv1_b1(int B, int n_lin, const int64_t* Ns, int64_t K, int rotate, float* ks_part, uint32_t* ks_ctr,
                   B1Config* cfg, const char** why) {
  if (B != 1) {
    *why = "the one-launch B = 1 kernel takes one token";
    return false;
  }
  const int BT = B == 1 ? 1 : B <= 4 ? 4 : B <= 8 ? 8 : 16;
  const int NSET = (BT + 3) / 4, NCOL = BT == 1 ? 2 : 8;
  if (n_lin < 1 || n_lin > GEMV_MAX_LIN) {
    *why = "1..4 linears per decode launch";
    return false;
  }
  const int G = static_cast<int>(K / 128);
  if (G < 1) {
    *why = "K must be a positive multiple of 128";
    return false;
  }
  B1Config c{};
  B1Args& a = c.a;
  double wbytes = 0;
  int CL = b1_cluster_size(n_lin, Ns, K, &wbytes);
  int KS = ks_part && ks_ctr ? b1_ks_slices(n_lin, Ns, K) : 1;
  if (KS > 1) CL = 2;
  const int NW = B1_NW;
  int TPS = std::max(1, std::min(64, b1_env("PARO_G1_TPS", 2 * NW)));
  const int threads = (NW + 1) * 32;
  c.NW = NW;
  const int budget = device_smem_optin() - 1024;
  // clusters that fit in one wave (occupancy API, cached per cluster size)
  int ncl_max = b1_active_clusters(BT, CL, threads, budget);
  ncl_max = std::min(ncl_max, std::max(1, b1_env("PARO_G1_MAXCL", 1 << 20)));
  // short multi-linear launches (q/k/v: < 20 MB over several linears): three quarters of the
  // clusters -- each CTA streams a longer run of tiles, and the SMs left free take the NEXT launch's
  // CTAs early (PDL: they fill their rings while this launch finishes).  Measured on the LLaMA-3-8B
  // step (same box, tools/ab_knobs.sh): q/k/v 6.77 -> 6.42 us, step 34.64 -> 34.15 us; 20 / 16 / 12 /
  // 8 clusters and single-linear launches (o_proj) measured slower.
  if (PARO_B1_SHORT_MULTI_CAP && n_lin > 1 && wbytes < 20e6) ncl_max = std::max(n_lin, ncl_max * 3 / 4);
  if (wbytes < 20e6) ncl_max = std::min(ncl_max, std::max(1, b1_env("PARO_G1_SMALL_MAXCL", 1 << 20)));
  // clusters over linears in proportion to their row blocks (>= 1 each, <= row blocks)
  int64_t NB[GEMV_MAX_LIN], NBsum = 0;
  for (int i = 0; i < n_lin; ++i) {
    NB[i] = (Ns[i] + TILE_ROWS - 1) / TILE_ROWS;
    NBsum += NB[i];
  }
  if (KS > 1) ncl_max /= KS;  // row ranges (each KS clusters)
  int ncl = static_cast<int>(std::min<int64_t>(ncl_max, NBsum));
  if (ncl < n_lin) ncl = n_lin;
  int cls[GEMV_MAX_LIN], used = 0, big = 0;
  for (int i = 0; i < n_lin; ++i) {
    cls[i] = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(NB[i], ncl * NB[i] / NBsum)));
    used += cls[i];
    if (NB[i] > NB[big]) big = i;
  }
  cls[big] = static_cast<int>(std::min<int64_t>(NB[big], cls[big] + std::max(0, ncl - used)));
  int begin = 0, rmax = 0;
  for (int i = 0; i < n_lin; ++i) {
    B1Linear& d = a.lin[i];
    d.N = static_cast<int>(Ns[i]);
    d.cta_begin = begin;
    d.rb_base = static_cast<int>(NB[i] / cls[i]);
    d.rb_extra = static_cast<int>(NB[i] % cls[i]);
    rmax = std::max(rmax, (d.rb_base + (d.rb_extra ? 1 : 0)) * TILE_ROWS);
    begin += cls[i] * CL * KS;
  }
  c.grid = begin;
  a.KS = KS;
  a.ks_part = KS > 1 ? ks_part : nullptr;
  a.ks_ctr = KS > 1 ? ks_ctr : nullptr;
  c.CL = CL;
  c.BT = BT;
  a.B = B;
  a.n_lin = n_lin;
  a.K = static_cast<int>(K);
  a.G = G;
  a.rotate = rotate;
  a.TPS = TPS;
  a.pre_stages = std::max(0, b1_env("PARO_G1_PRE", 2));
  a.params_first = b1_env("PARO_G1_PF", 1);
  a.R_max = rmax;
  a.RRmax = (rmax + CL - 1) / CL;
  const int gcm = ((G + KS - 1) / KS + CL - 1) / CL;
  a.sc_off = static_cast<uint32_t>(TPS) * TILE_CODE_BYTES;
  a.z_off = a.sc_off + static_cast<uint32_t>(TPS) * TILE_SCALE_BYTES;
  a.slot_bytes = b1_align(a.z_off + static_cast<uint32_t>(TPS) * TILE_ZERO_BYTES, 128);
  uint32_t off = 0;
  a.off_xp = off;
  off += b1_align(static_cast<uint32_t>(gcm) * NSET * 4 * NCOL * 32, 128);
  a.off_xs = off;
  off += b1_align(static_cast<uint32_t>(gcm) * BT * 8 + 48, 128);  // + a 16-aligned 32-byte zero block
  a.off_part = off;
  // B = 1: per-warp row partials summed in a fixed order (deterministic) while they fit in
  // 48 KB; clusters with more rows (e.g. 70B gate+up: 3840 rows) add with shared atomics
  // (K split: up to 64 KB, so that its row ranges of ~26 row blocks keep the deterministic sums)
  a.atom = BT == 1 && (static_cast<int64_t>(NW) * rmax * 4 > (b1_env("PARO_G1_ATOM_KB", KS > 1 ? 64 : 48) << 10));
  off += b1_align(static_cast<uint32_t>(BT == 1 && !a.atom ? NW : BT) * rmax * 4, 128);
  a.off_scr = a.off_recv = off;  // BT > 1: phase-1 scratch and the cluster reduction share this space
  if (BT == 1) {
    off += NW * 512;
    a.off_recv = off;
    off += b1_align(static_cast<uint32_t>(CL) * a.RRmax * 4, 128);
  } else {  // the transform runs in paro_gemv1_xform_kernel: no scratch
    off += b1_align(static_cast<uint32_t>(CL) * a.RRmax * BT * 4, 128);
  }
  a.off_bar = off;
  off += 64 * 16;
  a.off_ring = b1_align(off, 1024);
  const int64_t avail = static_cast<int64_t>(budget) - a.off_ring;
  // stage size: the largest TPS <= 32 (two tiles per warp) that keeps >= 2 stages in flight, else
  // the largest that fits once (stages a CTA needs: ceil(row blocks x groups / TPS)); measured
  // flat between 24 and 32 tiles per stage with 2-3 stages (tools/run_g1n.sh)
  const int64_t cta_tiles = static_cast<int64_t>(rmax / TILE_ROWS) * gcm;
  auto slot_of = [&](int tps) {
    const uint32_t sc = static_cast<uint32_t>(tps) * TILE_CODE_BYTES;
    return b1_align(sc + static_cast<uint32_t>(tps) * (TILE_SCALE_BYTES + TILE_ZERO_BYTES), 128);
  };
  auto stages_of = [&](int tps) {
    const int need = static_cast<int>((cta_tiles + tps - 1) / tps);
    return std::min<int64_t>(std::min(need, 60), avail / slot_of(tps));
  };
  if (b1_env("PARO_G1_TPS", 0) == 0) {
    int best = 0;
    for (int want = 2; want >= 1 && !best; --want)
      for (int tps = 2 * NW; tps >= 8 && !best; tps -= 4)
        if (stages_of(tps) >= std::min<int64_t>(want, (cta_tiles + tps - 1) / tps)) best = tps;
    TPS = best ? best : 8;
    // long-K launches (few groups per CTA in rows, many tiles): a third ring slot of 28 tiles beats
    // two of 32 (LLaMA-3-8B down_proj 10.3 -> 9.7 us, same box, tools/ab_knobs.sh)
    if (G >= 64 && TPS == 32 && stages_of(28) >= 3 && stages_of(32) < 3) TPS = 28;
  }
  a.TPS = TPS;
  a.sc_off = static_cast<uint32_t>(TPS) * TILE_CODE_BYTES;
  a.z_off = a.sc_off + static_cast<uint32_t>(TPS) * TILE_SCALE_BYTES;
  a.slot_bytes = slot_of(TPS);
  int S = static_cast<int>(stages_of(TPS));
  if (S < 1) {
    *why = "decode shared-memory plan does not fit";
    return false;
  }
  a.S = S;
  a.smem_total = a.off_ring + static_cast<uint32_t>(S) * a.slot_bytes;
  if (b1_env("PARO_PLAN_DEBUG", 0))
    fprintf(stderr, "[paro gemv1 plan] B=%d BT=%d n_lin=%d K=%lld grid=%d CL=%d NW=%d TPS=%d S=%d R_max=%d smem=%u\n",
            B, BT, n_lin, static_cast<long long>(K), c.grid, CL, NW, TPS, S, rmax, a.smem_total);
  *cfg = c;
  return true;
}

template <int BT>
static cudaError_t b1_launch(const B1Config& c, cudaLaunchConfig_t* cfg) {
  const bool at = c.a.atom != 0;
  auto kern = c.a.p2p  ? (at ? paro_gemv1_b1_kernel<B1_NW, BT, 2, true> : paro_gemv1_b1_kernel<B1_NW, BT, 2, false>)
              : c.a.KS > 1 ? (at ? paro_gemv1_b1_kernel<B1_NW, BT, 1, true> : paro_gemv1_b1_kernel<B1_NW, BT, 1, false>)
                           : (at ? paro_gemv1_b1_kernel<B1_NW, BT, 0, true> : paro_gemv1_b1_kernel<B1_NW, BT, 0, false>);
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), static_cast<int>(c.a.smem_total));
  if (e != cudaSuccess) return e;
  return cudaLaunchKernelEx(cfg, kern, c.a);
}

cudaError_t launch_gemv1_b1(const B1Config& c, cudaStream_t st) {
#if PARO_TIMELINE
  const_cast<B1Config&>(c).a.tl_slot = g_b1_seq++ & 15;
#endif
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(c.grid);
  cfg.blockDim = dim3((c.NW + 1) * 32);
  cfg.dynamicSmemBytes = c.a.smem_total;
  cfg.stream = st;
  cudaLaunchAttribute attrs[2];
  int na = 0;
  attrs[na].id = cudaLaunchAttributeClusterDimension;
  attrs[na].val.clusterDim.x = c.CL;
  attrs[na].val.clusterDim.y = 1;
  attrs[na].val.clusterDim.z = 1;
  ++na;
  if (c.a.pdl) {
    attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attrs;
  cfg.numAttrs = na;
  switch (c.BT) {
    case 1: return b1_launch<1>(c, &cfg);
    default: return cudaErrorInvalidConfiguration;
  }
}

}  // namespace paro
