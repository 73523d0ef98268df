// gemv1.cu -- decode path: scale + L Givens layers + group-wise INT4 dequant GEMV, as a
// PERSISTENT CHAIN of stages in one launch (a stage = one multi-linear GEMV whose linears share
// x; a single paro_linear / paro_linear_multi call is a one-stage chain).
//
// SURVEY.md 8(a) rows a4 (u = s . x), a5 (the L rotations, Eq. 5 in column
// form), a6 (dequant GEMV, Eq. 1 dequantisation (q - z) * S),
// a8 (bias + output rounding, Eq. 2); SURVEY.md 8(f) NEXT #1 (fused multi-linear
// launches chained without a kernel boundary).
//
// Work split (K-split inside a thread-block cluster), per stage:
//  * a cluster of CL CTAs (one per SM, one wave) owns a run of 32-row blocks of one linear;
//  * CTA c of the cluster owns the groups [c G / CL, (c + 1) G / CL) of those rows.  It
//    transforms ONLY its own groups (a warp per group: the rotation is group-local, so no
//    activation ever crosses CTAs) and streams only the tiles of its groups;
//  * the cluster sums its CTAs' row partials through distributed shared memory (st.async,
//    fixed order) and the owner CTA of a row writes y.  Within a CTA, B = 1 keeps per-warp row
//    partials summed in a fixed order (deterministic) unless the cluster has too many rows;
//    B > 1 and those clusters use shared-memory atomics.
// Chain: stage s + 1 may read an earlier stage's y as its x, so every CTA passes a grid-wide
// barrier (all CTAs co-resident: one wave) after storing its stage-s rows and before loading
// stage s + 1's x.  The WEIGHTS never depend on earlier stages: one producer warp per CTA streams
// the tiles of all stages, back to back, through one cp.async.bulk (TMA engine) ring, so while a
// stage's dependent chain runs (reduction, store, barrier, x load, transform) the ring fills with
// the next stage's weights and the HBM stream does not stop at stage boundaries.  Stage 0's
// first batches go out before the programmatic-dependent-launch wait (packed weights are never
// written by the previous kernel); the rest once the compute warps' rotation parameters and x
// are requested, so those latency-critical loads do not queue behind the weight stream.
// B = 2..16: stage 0's x' digits of all tokens come from paro_gemv1_xform_kernel (once per
// (linear, group, four tokens)); later stages compute them inside the launch (every warp of the
// grid takes transform tasks, then one more grid barrier) -- the producer / thread 0
// bulk-copies each CTA's groups' slice.
//
// Dot product on the warp-level integer tensor cores (IMMA.16832, u8 x s8 -> s32, exact):
// x' of a group becomes 16-bit fixed point x'fix = rint(x' 2^(14 - E)) with 2^E >= max |x'|
// (|x'fix| <= 2^14), split into two s8 digits x'fix = 256 hi + lo.  An AND mask on a code word
// gives four u8 codes (low nibbles: q; high nibbles: 16 q), which ARE the A fragment of the
// MMA; B holds the digits (column 0: hi, column 1: lo).  Per (row, group) the int32 result
// I = sum (q - z) x'fix is exact and y += S * 2^(E - 14) * I.  Lane (g, t) of a warp loads
// quad t of rows g, g + 8, g + 16, g + 24 of a tile (four LDS.128, 128 weights); eight MMAs
// cover the tile.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "paro_internal.h"
#include "ptx.cuh"
#include "tile_layout.cuh"
#include "umma.cuh"

namespace paro {

#ifndef PARO_G1_MERGE_NIB
#define PARO_G1_MERGE_NIB 1  // B > 1 mma.sync tiles: low and high nibbles into one accumulator
#endif
#ifndef PARO_TIMELINE
#define PARO_TIMELINE 0  // 1: %globaltimer marks per (CTA, stage, event) for tools/timeline_chain.py
#endif
#if PARO_TIMELINE
__device__ unsigned long long g_tl[1024 * 16 * 8];
extern "C" int paro_debug_timeline(unsigned long long* host, int n) {
  if (n > 1024 * 16 * 8) n = 1024 * 16 * 8;
  return static_cast<int>(cudaMemcpyFromSymbol(host, g_tl, sizeof(unsigned long long) * n));
}
#endif
__device__ __forceinline__ void tl_mark(int s, int ev) {
#if PARO_TIMELINE
  if (blockIdx.x < 1024 && s < 16) g_tl[(blockIdx.x * 16 + s) * 8 + ev] = globaltimer_ns();
#else
  (void)s;
  (void)ev;
#endif
}

namespace {
// compute warps per CTA (+ 1 producer warp).  16 warps in all keep four warps per SM
// sub-partition and so 128 registers per thread (17 warps would cap it at 96 and spill); B > 1
// uses three warpgroups of four for the tensor-core tiles.
// B = 1 one-stage instances (no stage loop) fit 16 compute warps in 96 registers without spills;
// chain instances and B > 1 keep more live state and use 15 (16 warps in all: 128 registers), the
// tcgen05 engine three warpgroups.
__host__ __device__ constexpr int g1_nw(int BT, bool um, bool chain) {
  return BT > 1 ? (um ? 12 : 15) : (chain ? 15 : 16);
}
constexpr uint32_t TILE_B = TILE_CODE_BYTES + TILE_SCALE_BYTES + TILE_ZERO_BYTES;

// D(16x8 s32) += A(16x32 u8, row) * B(32x8 s8, col); fragments as in ptx.cuh (imma_16832),
// not volatile so the scheduler may interleave the four accumulator chains
__device__ __forceinline__ void mma_u8s8(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
  asm("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// This CTA's share of a stage.
struct G1Geom {
  int li;         // linear
  int active;     // the CTA has work in this stage
  int rb0, R;     // first row block, rows (cluster-wide)
  int ga, gc;     // first group, groups (this CTA's K-split share)
  int n_tiles, n_batches;
  int RR, my_lo, my_n;  // reduction: rows per owner CTA, my owned rows
  int nrb, nch;         // B > 1: row blocks; group chunks per row-block quad
};

// B = 1: a batch is TPS consecutive tiles of the sequence (row block, group).  B > 1: a batch
// is (row-block quad q, group chunk c): the tiles (4 q + j, gamma) for j < 4 and gamma in chunk
// c of TPS / 4 groups, stored j-major (the four row blocks of one group form one M = 128 MMA).
__device__ __forceinline__ G1Geom g1_geom(const Gemv1Stage& S, int lgCL, int crank, int TPS, bool quads) {
  G1Geom g{};
  const int bx = static_cast<int>(blockIdx.x);
  g.active = bx < S.n_cta;
  if (!g.active) return g;
  int li = 0;
#pragma unroll 1
  while (li + 1 < S.n_lin && bx >= S.lin[li + 1].cta_begin) ++li;
  g.li = li;
  const Gemv1Linear& d = S.lin[li];
  const int cl = (bx - d.cta_begin) >> lgCL;  // cluster sizes are powers of two
  const int nrb = d.rb_base + (cl < d.rb_extra ? 1 : 0);
  g.rb0 = cl * d.rb_base + min(cl, d.rb_extra);
  g.R = nrb * TILE_ROWS;
  g.ga = (crank * S.G) >> lgCL;
  g.gc = (((crank + 1) * S.G) >> lgCL) - g.ga;
  g.n_tiles = nrb * g.gc;
  g.nrb = nrb;
  if (quads) {
    const int m = TPS / 4;
    g.nch = (g.gc + m - 1) / m;
    g.n_batches = ((nrb + 3) / 4) * g.nch;
  } else {
    g.n_batches = (g.n_tiles + TPS - 1) / TPS;
  }
  g.RR = (g.R + (1 << lgCL) - 1) >> lgCL;
  g.my_lo = crank * g.RR;
  g.my_n = max(0, min(g.RR, g.R - g.my_lo));
  return g;
}

// x' of one group of one token chunk as fixed point + s8 digits laid out as the GEMV's B
// fragments [quad t][column][k-block kb][b0, b1]; column 2 cb + dg = digit dg (0 hi, 1 lo) of
// token cb of the column set; k-block kb = 2 p + h covers the low (p = 0) or high (p = 1)
// nibbles of words 2h, 2h + 1 (b0: word 2h, b1: word 2h + 1); byte bb of the word for quad t,
// word j, parity p is channel tile_k(t, j, 2 bb + p).  sc: the group's 128 rotated values
// (fp32, overwritten with x'fix).  Returns (sum x'fix, bits of 2^(E - 14)) in lane 0's result.
template <int NCOLS>
__device__ __forceinline__ int2 g1_digits(float* sc, int lane, uint8_t* dst_set, int cb) {
  int* fx = reinterpret_cast<int*>(sc);
  const float4 v = *reinterpret_cast<const float4*>(sc + 4 * lane);
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
  *reinterpret_cast<uint2*>(dst_set + tq * (NCOLS * 32) + (2 * cb + col) * 32 + kb * 8) = make_uint2(wd[0], wd[1]);
  return make_int2(X, static_cast<int>(static_cast<uint32_t>(113 + E) << 23));  // 2^(E - 14)
}

// a4 for TB tokens of one group: scr[tb][128] = s . x_tb
template <int TB>
__device__ __forceinline__ void g1_scale(float* scr, const uint2 (&xv)[TB], int x_bf16, float4 sv, int lane) {
#pragma unroll
  for (int tb = 0; tb < TB; ++tb) {
    float2 f01, f23;
    if (x_bf16) {
      f01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xv[tb].x));
      f23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xv[tb].y));
    } else {
      f01 = __half22float2(*reinterpret_cast<const __half2*>(&xv[tb].x));
      f23 = __half22float2(*reinterpret_cast<const __half2*>(&xv[tb].y));
    }
    *reinterpret_cast<float4*>(scr + tb * 128 + 4 * lane) =
        make_float4(f01.x * sv.x, f01.y * sv.y, f23.x * sv.z, f23.y * sv.w);
  }
  __syncwarp();
}

// a5 for TB tokens in lockstep: rotations t = 1..L, each pair from the pre-update values
// (Eq. 4 / Eq. 5); lane l updates the pairs of slots l and l + 32
template <int TB>
__device__ __forceinline__ void g1_rot(float* scr, const float4 (&cs)[8], const uint32_t (&ix)[8], int L) {
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
}

// rotation records [group][layer][32 lanes]: (cos, sin) of slots lane, lane + 32 and their
// (i, j) channel pairs (pack-time bank-conflict-free schedule), and s of the lane's 4 channels
__device__ __forceinline__ void g1_params(const Gemv1Linear& d, int gam, int L, int rotate, int lane, float4 (&cs)[8],
                                          uint32_t (&ix)[8], float4& sv) {
  const int64_t rec = static_cast<int64_t>(gam) * L * 32 + lane;
#pragma unroll
  for (int t = 0; t < 8; ++t)
    if (t < L) {
      cs[t] = __ldg(reinterpret_cast<const float4*>(d.rot_cs) + rec + t * 32);
      ix[t] = __ldg(reinterpret_cast<const uint32_t*>(d.rot_idx) + rec + t * 32);
    }
  sv = rotate ? __ldg(reinterpret_cast<const float4*>(d.svec + gam * 128) + lane) : make_float4(1.f, 1.f, 1.f, 1.f);
}

// x of token b, channels 4 lane .. 4 lane + 3 of group gam.  coherent: x may have been written
// earlier in this launch by another SM (a later chain stage): L2 load; else the read-only path.
__device__ __forceinline__ uint2 g1_ldx(const void* x, int64_t K, int b, int gam, int lane, bool coherent) {
  const uint2* p = reinterpret_cast<const uint2*>(static_cast<const uint8_t*>(x) +
                                                  (static_cast<int64_t>(b) * K + gam * 128 + 4 * lane) * 2);
  return coherent ? __ldcg(p) : __ldg(p);
}

// B > 1: x' of one (group, token) as fixed point + s8 digits in the UMMA B-operand layout of the
// group: rows n = 2 b (hi digit of token b) and 2 b + 1 (lo digit), 128 K-bytes each, K-major
// with the 128-byte swizzle (16-byte chunk c of row n at chunk c ^ (n % 8); 8-row groups 1024 B
// apart).  K index k < 64: byte k % 4 of the LOW-nibble word k / 4 of a tile row (channel
// tile_k(t, j, 2 bb) for word 4 t + j); k >= 64: the HIGH nibbles of word (k - 64) / 4.  The
// A operand (the masked code words, csrc/gemv1.cu phase 2) uses the same K order.
__device__ __forceinline__ int2 g1_digits_umma(float* sc, int lane, uint8_t* grp, int b) {
  int* fx = reinterpret_cast<int*>(sc);
  const float4 v = *reinterpret_cast<const float4*>(sc + 4 * lane);
  const float ml = fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w)));
  const uint32_t mb = __reduce_max_sync(0xffffffffu, __float_as_uint(ml));
  int E = mb < 0x00800000u ? -100 : static_cast<int>(mb >> 23) - 127 + ((mb & 0x7fffffu) != 0u ? 1 : 0);
  E = max(E, -100);
  const float mul = __uint_as_float(static_cast<uint32_t>(141 - E) << 23);  // 2^(14 - E)
  const int f0 = __float2int_rn(v.x * mul), f1 = __float2int_rn(v.y * mul);
  const int f2 = __float2int_rn(v.z * mul), f3 = __float2int_rn(v.w * mul);
  const int X = __reduce_add_sync(0xffffffffu, (f0 + f1) + (f2 + f3));
  __syncwarp();
  *reinterpret_cast<int4*>(fx + 4 * lane) = make_int4(f0, f1, f2, f3);
  __syncwarp();
  const int w = lane & 15, t = w >> 2, j = w & 3, p = lane >> 4;
  uint32_t whi = 0, wlo = 0;
#pragma unroll
  for (int bb = 0; bb < 4; ++bb) {
    const int c = 32 * j + 16 * p + 2 * t + (bb >> 1) + 8 * (bb & 1);  // tile_k(t, j, 2 bb + p)
    const int f = fx[c];
    const int lo = static_cast<int>(static_cast<int8_t>(f & 0xff));
    whi |= (static_cast<uint32_t>((f - lo) >> 8) & 0xffu) << (8 * bb);
    wlo |= (static_cast<uint32_t>(lo) & 0xffu) << (8 * bb);
  }
  const int nh = 2 * b, nl = 2 * b + 1;
  *reinterpret_cast<uint32_t*>(grp + (nh >> 3) * 1024 + (nh & 7) * 128 + (((lane >> 2) ^ (nh & 7)) << 4) +
                               4 * (lane & 3)) = whi;
  *reinterpret_cast<uint32_t*>(grp + (nl >> 3) * 1024 + (nl & 7) * 128 + (((lane >> 2) ^ (nl & 7)) << 4) +
                               4 * (lane & 3)) = wlo;
  return make_int2(X, static_cast<int>(static_cast<uint32_t>(113 + E) << 23));  // 2^(E - 14)
}

// B > 1: one transform task = (linear, group, token) -> digits + (sum, scale) in the linear's
// xq / xqs buffers (the layout the GEMV bulk-copies).  One token per warp: the tasks are
// independent, so the transform's latency (it sits between two dependent GEMV launches) is that
// of one token's 8 rotations, not four tokens' in lockstep.  Tokens B .. BT - 1 get x = 0.
template <int BT, bool UM>
__device__ __forceinline__ void g1_xform_task(const Gemv1Stage& S, int task, int B, int x_bf16, int rotate, float* scr,
                                              int lane, bool wait_pdl) {
  constexpr int NB = BT / 4, XPC = 4 * 8 * 32, XPG = NB * XPC;  // = 2 BT rows x 128 B (UMMA B tile)
  const int G = S.G;
  const int li = task / (G * BT), rem = task - li * G * BT, gam = rem / BT, b = rem - gam * BT;
  const Gemv1Linear& d = S.lin[li];
  const int L = rotate ? d.L : 0;
  float4 cs[8], sv;
  uint32_t ix[8];
  g1_params(d, gam, L, rotate, lane, cs, ix, sv);
  if (wait_pdl) pdl_wait();  // x may be written by the previous kernel on the stream
  uint2 xv[1] = {b < B ? g1_ldx(S.x, S.K, b, gam, lane, !wait_pdl) : make_uint2(0u, 0u)};
  g1_scale<1>(scr, xv, x_bf16, sv, lane);
  g1_rot<1>(scr, cs, ix, L);
  uint8_t* xq = d.xq + static_cast<size_t>(gam) * XPG;
  // tcgen05 engine: the group's UMMA B tile; mma.sync engine: the column set's B fragments
  const int2 r = UM ? g1_digits_umma(scr, lane, xq, b) : g1_digits<8>(scr, lane, xq + (b >> 2) * XPC, b & 3);
  if (lane == 0) d.xqs[static_cast<size_t>(gam) * BT + b] = r;
}

}  // namespace

// NW compute warps + 1 producer warp (17 warps: up to 96 registers per thread).
// BT: token capacity of the instance (1, 4, 8, 16).  MS: stage capacity of the argument block.
// UM_: B > 1 tiles on the tcgen05 tensor cores (kind::i8, TMEM) instead of warp-level mma.sync.
// B > 1 single launches leave one paro_gemv1_xform_kernel CTA's registers (128 threads x 64) and
// shared memory free on every SM (PARO_G1_COXFORM): the NEXT launch's pre-kernel then runs beside
// this GEMV's CTAs instead of holding the next GEMV's CTAs (and so its weight stream) back.
#ifndef PARO_G1_COXFORM
#define PARO_G1_COXFORM 1
#endif
template <int NW, int BT, int MS, bool UM_>
__global__ void __launch_bounds__((NW + 1) * 32, 1)
    __maxnreg__((PARO_G1_COXFORM && BT == 16 && MS == 1) ? 112 : 128)
    paro_gemv1_kernel(const __grid_constant__ Gemv1ArgsT<MS> a);
template <int NW, int BT, int MS, bool UM_>
__global__ void __launch_bounds__((NW + 1) * 32, 1)
    __maxnreg__((PARO_G1_COXFORM && BT == 16 && MS == 1) ? 112 : 128)
    paro_gemv1_kernel(const __grid_constant__ Gemv1ArgsT<MS> a) {
  constexpr bool UM = BT > 1 && UM_;
  constexpr int TB = BT == 1 ? 1 : 4;          // tokens per MMA column set
  constexpr int NB = (BT + 3) / 4;             // column sets
  constexpr int NCOL = BT == 1 ? 2 : 8;        // B columns holding digits
  constexpr int XTQ = NCOL * 32;               // digit bytes per (group, set, quad)
  constexpr int XPC = 4 * XTQ;                 // digit bytes per (group, column set)
  constexpr int XPG = NB * XPC;                // digit bytes per group
  (void)TB;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  // 1024-byte aligned base (the UMMA B tiles use the 128-byte swizzle); the plan reserves the slack
  // tcgen05 engine: 1024-byte aligned base (the UMMA B tiles use the 128-byte swizzle; the plan
  // reserves the slack)
  uint8_t* smem = UM ? smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u) : smem_raw;
  static_assert(NW % 4 == 0 || !UM, "the tcgen05 engine needs whole warpgroups");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int CL = static_cast<int>(cluster_nctarank());
  const int crank = static_cast<int>(cluster_ctarank());
  const int B = a.B;
  const int n_st = MS == 1 ? 1 : a.n_stages;  // a one-stage instance has no stage loop

  uint8_t* xp = smem + a.off_xp;                                 // x' digits [gc][NB][4 t][NCOL][4 kb][8 B]
  int2* xs = reinterpret_cast<int2*>(smem + a.off_xs);           // per (group, token): (sum x'fix, 2^(E-14))
  const uint8_t* zblk = smem + a.off_xs - 32;                    // 32 zero bytes (B columns >= 2)
  float* part = reinterpret_cast<float*>(smem + a.off_part);     // BT = 1: [NW][R_max]; else [R_max][BT]
  float* recv = reinterpret_cast<float*>(smem + a.off_recv);     // [CL][RRmax][BT] cluster partials
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.off_bar);
  uint64_t* empty = full + a.S;
  uint64_t* rbar = empty + a.S;  // cluster partials of my rows landed (st.async bytes), one phase per stage
  uint64_t* xbar = rbar + 1;     // BT > 1: the pre-transformed x' slice landed
  uint64_t* mdone = xbar + 1;    // BT > 1: [warpgroup][2 buffers] the MMAs completed (tcgen05.commit)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mdone + 8);  // BT > 1: TMEM base address
  uint8_t* ring = smem + a.off_ring;
  // this CTA's share of every stage (read from shared memory where used: keeps registers free);
  // the stages' shares are computed in parallel by threads 0 .. n_stages - 1 while warp 1 sets up
  // the barriers (nothing serial on the launch's critical path)
  __shared__ G1Geom sgeo[MS];
  const int lgCL = __ffs(CL) - 1;
  if (tid < n_st) sgeo[tid] = g1_geom(a.st[tid], lgCL, crank, a.TPS, UM);

  if (tid < 8) reinterpret_cast<uint32_t*>(smem + a.off_xs - 32)[tid] = 0u;
  // barrier initialisation spread over threads 32 .. (each init is a store plus an async-proxy
  // fence: done serially by one thread it sits on the launch's critical path)
  if (tid >= 32 && tid < 32 + a.S) {
    mbar_init(&full[tid - 32], 1);
    mbar_init(&empty[tid - 32], NW);
    fence_mbar_init();
  } else if (tid >= 96 && tid < 106) {
    if (tid < 104)
      mbar_init(&mdone[tid - 96], 1);
    else
      mbar_init(tid == 104 ? rbar : xbar, 1);
    fence_mbar_init();
  }
  if (UM && warp == 2) tmem_alloc(tmem_slot, 512);  // 3 warpgroups x (2 A + 2 D buffers) <= 512 columns
  if constexpr (UM) tc_fence_before();
  __syncthreads();
  if constexpr (UM) tc_fence_after();
  // stage 0's cluster partials of my rows (the arm may follow remote bytes: the phase cannot
  // complete before this arrival)
  if (tid == 0 && CL > 1) mbar_arrive_expect_tx(rbar, static_cast<uint32_t>((CL - 1) * sgeo[0].my_n * BT * 4));
  if (tid == 0) tl_mark(0, 0);
  if (CL > 1) cluster_arrive_relaxed();  // every CTA's mbarriers are initialised (DSMEM legal after the wait)
  if (a.pdl) pdl_launch_dependents();

  // ------------------------------------------------------------ producer warp: the whole ring, every stage
  if (warp == NW) {
    const uint64_t pol = l2_evict_first_policy();
    const int pre = a.pre_stages;
    bool released = false;
    auto release = [&](const Gemv1Stage& S, const G1Geom& g) {
      // stage 0, B > 1: x' digits of my groups, written by the preceding xform kernel
      if (BT > 1 && g.active) {
        if (a.pdl) pdl_wait();
        if (lane == 0) {
          const Gemv1Linear& d = S.lin[g.li];
          const uint32_t nd = static_cast<uint32_t>(g.gc * XPG), ns = static_cast<uint32_t>(g.gc * BT * 8);
          mbar_arrive_expect_tx(xbar, nd + ns);
          bulk_g2s_nohint(xp, d.xq + static_cast<size_t>(g.ga) * XPG, nd, xbar);
          bulk_g2s_nohint(xs, d.xqs + static_cast<size_t>(g.ga) * BT, ns, xbar);
        }
        __syncwarp();
      }
      named_bar_sync(2, (NW + 1) * 32);  // the compute warps' x / parameter loads are out
      released = true;
    };
    if (a.params_first) named_bar_sync(3, (NW + 1) * 32);  // the rotation-parameter loads are out
    // the segments of batch bt of a stage: bulk copies into a ring slot, or L2 prefetches (dst NULL)
    auto batch = [&](const G1Geom& g, const Gemv1Linear& d, int G, int bt, uint8_t* dst, uint64_t* bar) {
      auto seg = [&](uint32_t i0, int64_t T, uint32_t n) {
        if (dst) {
          bulk_g2s(dst + i0 * TILE_CODE_BYTES, d.codes + T * TILE_CODE_BYTES, n * TILE_CODE_BYTES, bar, pol);
          bulk_g2s(dst + a.sc_off + i0 * TILE_SCALE_BYTES, d.scales + T * TILE_SCALE_BYTES, n * TILE_SCALE_BYTES,
                   bar, pol);
          bulk_g2s(dst + a.z_off + i0 * TILE_ZERO_BYTES, d.zeros + T * TILE_ZERO_BYTES, n * TILE_ZERO_BYTES, bar,
                   pol);
        } else {
          prefetch_l2_bulk(d.codes + T * TILE_CODE_BYTES, n * TILE_CODE_BYTES);
          prefetch_l2_bulk(d.scales + T * TILE_SCALE_BYTES, n * TILE_SCALE_BYTES);
          prefetch_l2_bulk(d.zeros + T * TILE_ZERO_BYTES, n * TILE_ZERO_BYTES);
        }
      };
      if constexpr (!UM) {
        const int u0 = bt * a.TPS, u1 = min(g.n_tiles, u0 + a.TPS);
        if (dst) mbar_arrive_expect_tx(bar, static_cast<uint32_t>(u1 - u0) * TILE_B);
#pragma unroll 1
        for (int u = u0; u < u1;) {  // one contiguous segment per row block touched
          const int rb = u / g.gc, ue = min(u1, (rb + 1) * g.gc);
          seg(static_cast<uint32_t>(u - u0), static_cast<int64_t>(g.rb0 + rb) * G + g.ga + (u - rb * g.gc),
              static_cast<uint32_t>(ue - u));
          u = ue;
        }
      } else {
        // (quad q, chunk c): one contiguous segment of mm tiles per row block 4 q + j
        const int m = a.TPS / 4, q = bt / g.nch, c = bt - q * g.nch;
        const int mm = min(m, g.gc - c * m), nq = min(4, g.nrb - 4 * q);
        if (dst) mbar_arrive_expect_tx(bar, static_cast<uint32_t>(nq * mm) * TILE_B);
#pragma unroll 1
        for (int j = 0; j < nq; ++j)
          seg(static_cast<uint32_t>(j * mm), static_cast<int64_t>(g.rb0 + 4 * q + j) * G + g.ga + c * m,
              static_cast<uint32_t>(mm));
      }
    };
    int slot = 0, phase = 0, nb = 0;
#pragma unroll 1
    for (int s = 0; s < n_st; ++s) {
      const Gemv1Stage& S = a.st[s];
      const G1Geom& g = sgeo[s];
      const Gemv1Linear& d = S.lin[g.li];
      const int G = S.G;
      if (s > 0) {
        // Stage boundary.  The ring drains while the compute warps finish stage s - 1, pass the
        // grid barrier and load this stage's x: bulk copies issued now would sit in front of
        // those latency-critical loads (an SM's requests are served in order), so this stage's
        // first batches go to L2 as prefetches (no data returns to the SM), and the ring refill
        // -- from L2 -- starts once the compute warps' x loads are out.
        if (lane == 0)
          for (int bt = 0; bt < min(g.n_batches, a.l2_batches); ++bt) batch(g, d, G, bt, nullptr, nullptr);
        __syncwarp();
        if (a.xfirst) named_bar_sync(2, (NW + 1) * 32);
      }
#pragma unroll 1
      for (int bt = 0; bt < g.n_batches; ++bt) {
        if (s == 0 && bt == pre) release(S, g);
        if (nb >= a.S) mbar_wait(&empty[slot], phase ^ 1);
        if (lane == 0) batch(g, d, G, bt, ring + static_cast<size_t>(slot) * a.slot_bytes, &full[slot]);
        __syncwarp();
        ++nb;
        if (++slot == a.S) {
          slot = 0;
          phase ^= 1;
        }
      }
      if (lane == 0) tl_mark(s, 7);
      if (s == 0 && !released) release(S, g);
    }
    if (CL > 1) cluster_wait();
    return;
  }

  // ------------------------------------------------------------ compute warps
  int slot = 0, phase = 0, xuse = 0;
  uint32_t mma_it = 0;  // BT > 1: this warpgroup's MMA items so far (buffer and barrier parity; continues across stages)
  // grid barrier: warp 0 knows the launch epoch (64 e); every compute thread counts barriers
  const GridBar gb{a.gbar, a.gbar + 16};
  uint32_t ep = 0;
  uint32_t nbar = 0;
  auto arrive_grid = [&]() {  // after a CTA barrier over the compute warps
    ++nbar;
    if (tid == 0) grid_arrive(gb, ep + nbar);
  };
  auto wait_grid = [&]() {
    if (warp == 0 && !a.nobar) grid_wait_warp(gb, ep + nbar, lane);
    // reached from different call sites (per warp) after lanes left the poll loop apart: the
    // non-.aligned barrier form
    named_bar_sync_na(4, NW * 32);
  };
#pragma unroll 1
  for (int s = 0; s < n_st; ++s) {
    const Gemv1Stage& S = a.st[s];
    const G1Geom& g = sgeo[s];
    const Gemv1Linear& d = S.lin[g.li];
    const int ga = g.ga, gc = g.gc;
    float* pw = part + static_cast<size_t>(warp) * S.R_max;
    if (g.active) {
      if (BT == 1 && !S.atom) {
        for (int i = lane; i < g.R; i += 32) pw[i] = 0.f;
      } else {
        for (int i = tid; i < g.R * BT; i += NW * 32) part[i] = 0.f;
      }
    }

    // ---------------------------------------------------------- phase 1: x' of my groups (a4, a5)
    if constexpr (BT > 1) {
      if (s == 0) {
        if (a.params_first) named_bar_arrive(3, (NW + 1) * 32);
        named_bar_arrive(2, (NW + 1) * 32);
        if (a.pdl) pdl_wait();
        if (warp == 0 && n_st > 1) ep = ld_relaxed_gpu(gb.epoch) << 6;
      } else {
        wait_grid();
        if (S.xq_in_kernel) {
          // this stage's x is an earlier stage's y: transform tasks over every warp of the grid,
          // then one more grid barrier before the slices are copied
          float* scr = reinterpret_cast<float*>(smem + a.off_scr) + warp * 128;
          const int n_tasks = S.n_lin * S.G * BT;
#pragma unroll 1
          for (int task = static_cast<int>(blockIdx.x) * NW + warp; task < n_tasks;
               task += static_cast<int>(gridDim.x) * NW)
            g1_xform_task<BT, UM>(S, task, B, a.x_bf16, a.rotate, scr, lane, false);
          asm volatile("fence.proxy.async.global;" ::: "memory");  // generic writes -> bulk-copy reads
          named_bar_sync(1, NW * 32);
          arrive_grid();
          wait_grid();
        }
        if (g.active && tid == 0) {
          const uint32_t nd = static_cast<uint32_t>(gc * XPG), ns = static_cast<uint32_t>(gc * BT * 8);
          mbar_arrive_expect_tx(xbar, nd + ns);
          bulk_g2s_nohint(xp, d.xq + static_cast<size_t>(ga) * XPG, nd, xbar);
          bulk_g2s_nohint(xs, d.xqs + static_cast<size_t>(ga) * BT, ns, xbar);
        }
        if (a.xfirst) named_bar_arrive(2, (NW + 1) * 32);  // the x' slice is requested: the ring refill may start
      }
      if (g.active) {
        mbar_wait(xbar, xuse & 1);
        ++xuse;
      }
      if (tid == 0) tl_mark(s, 1);
    } else {
      float* scr = reinterpret_cast<float*>(smem + a.off_scr) + warp * 128;
      const int L = a.rotate ? d.L : 0;
      const bool mine = g.active && warp < gc;
      if (mine && lane == 0) {
        // later rounds' rotation records -> L2 now, ahead of the weight stream
        for (int gg = warp + NW; gg < gc; gg += NW) {
          const int64_t rec = static_cast<int64_t>(ga + gg) * L * 32;
          if (L > 0) {
            prefetch_l2_bulk(reinterpret_cast<const float4*>(d.rot_cs) + rec, static_cast<uint32_t>(L * 32 * 16));
            prefetch_l2_bulk(reinterpret_cast<const uint32_t*>(d.rot_idx) + rec, static_cast<uint32_t>(L * 32 * 4));
          }
          if (a.rotate) prefetch_l2_bulk(d.svec + (ga + gg) * 128, 512u);
        }
      }
      // the x dependency: the previous kernel on the stream (stage 0, PDL) or the previous stage
      // (grid barrier) -- waited for once the first group's rotation parameters are requested
      bool waited = false, arrived = s != 0 && !a.xfirst;
      auto wait_x = [&]() {
        if (s == 0) {
          if (a.params_first) {
            __syncwarp();
            named_bar_arrive(3, (NW + 1) * 32);
          }
          if (a.pdl) pdl_wait();
          if (warp == 0 && n_st > 1) ep = ld_relaxed_gpu(gb.epoch) << 6;
        } else {
          wait_grid();
        }
        if (tid == 0) tl_mark(s, 1);
        waited = true;
      };
#pragma unroll 1
      for (int gg = warp; mine && gg < gc; gg += NW) {
        const int gam = ga + gg;
        float4 cs[8], sv;
        uint32_t ix[8];
        g1_params(d, gam, L, a.rotate, lane, cs, ix, sv);
        if (!waited) wait_x();
        uint2 xv[1] = {g1_ldx(S.x, S.K, 0, gam, lane, s != 0)};
        g1_scale<1>(scr, xv, a.x_bf16, sv, lane);
        if (!arrived) {
          named_bar_arrive(2, (NW + 1) * 32);  // my x and parameters are in
          arrived = true;
        }
        g1_rot<1>(scr, cs, ix, L);
        const int2 r = g1_digits<NCOL>(scr, lane, xp + gg * XPG, 0);
        if (lane == 0) xs[gg] = r;
        __syncwarp();
      }
      if (!waited) wait_x();
      if (!arrived) named_bar_arrive(2, (NW + 1) * 32);
    }
    named_bar_sync(1, NW * 32);  // every x' of the CTA is in shared memory (and part zeroed)
    if (tid == 0) tl_mark(s, 2);

    // ---------------------------------------------------------- phase 2: tiles (a6)
    if constexpr (BT == 1) {
      const int gq = lane >> 2, tq = lane & 3;
      const bool atom = S.atom != 0;
      // batch bookkeeping advanced incrementally (no divisions in the loop): first tile of the
      // batch u0 = bt * TPS = r_lo * gc + off0
      int r_lo = 0, off0 = 0;
#pragma unroll 1
      for (int bt = 0; bt < g.n_batches; ++bt) {
        // batch tiles [u0, u1): tile i is (row block r_lo + ri, group ga + gi) with (ri, gi) = divmod(off0 + i, gc)
        const int u0 = bt * a.TPS, nt = min(g.n_tiles, u0 + a.TPS) - u0;
        mbar_wait(&full[slot], phase);
        if (bt == 0 && tid == 0) tl_mark(s, 3);
        const uint8_t* sb = ring + static_cast<size_t>(slot) * a.slot_bytes;
        int ri = 0, gi = off0 + warp;  // tile warp + k NW of the batch
        while (gi >= gc) {
          gi -= gc;
          ++ri;
        }
#pragma unroll 1
        for (int i = warp; i < nt; i += NW) {
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
          // B fragments: lanes of MMA columns >= 2 read a 32-byte zero block (address select, no branch)
          const uint8_t* bp = gq < 2 ? xp + gi * XPG + tq * XTQ + gq * 32 : zblk;
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
          // lane (gq, tq) holds columns 2 tq (hi digit) and 2 tq + 1 (lo digit); column pair 0 = the token
          if (tq == 0) {
            const int2 xf = xs[gi];
            const float F = __int_as_float(xf.y);
            float out[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int hh = q >> 1, e = (q & 1) * 2;
              const int zq = static_cast<int>((zw >> (4 * q)) & 15u);
              const int I = Dl[hh][e] * 256 + Dl[hh][e + 1] + ((Dh[hh][e] * 256 + Dh[hh][e + 1]) >> 4) - zq * xf.x;
              out[q] = Sr[q] * F * static_cast<float>(I);
            }
            if (!atom) {  // one uniform branch per tile, not per row
#pragma unroll
              for (int q = 0; q < 4; ++q) pw[rowl + 8 * q] += out[q];
            } else {
#pragma unroll
              for (int q = 0; q < 4; ++q) atomicAdd(part + rowl + 8 * q, out[q]);
            }
          }
          gi += NW;
          while (gi >= gc) {
            gi -= gc;
            ++ri;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
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
    } else if constexpr (!UM) {
      // B > 1 on the warp-level integer tensor cores: warp w takes a contiguous chunk of the batch's
      // tiles (row block ri, group gi), so that its consecutive tiles mostly share a row block and
      // the row partials (shared-memory atomics) are added once per row block; column sets of four
      // tokens (hi / lo digits in the MMA's 8 columns).  (Measured: plain per-warp partial slots
      // summed after each batch instead of the atomics -- no faster; the batch loop is latency-bound.)
      const int gq = lane >> 2, tq = lane & 3;
      int r_lo = 0, off0 = 0;
#pragma unroll 1
      for (int bt = 0; bt < g.n_batches; ++bt) {
        const int u0 = bt * a.TPS, nt = min(g.n_tiles, u0 + a.TPS) - u0;
        mbar_wait(&full[slot], phase);
        if (bt == 0 && tid == 0) tl_mark(s, 3);
        const uint8_t* sb = ring + static_cast<size_t>(slot) * a.slot_bytes;
        const int per = (nt + NW - 1) / NW;
        const int i_end = min(nt, (warp + 1) * per);
        int i = warp * per;
        int ri = (off0 + i) / gc, gi = off0 + i - ri * gc;
        float acc[NB][4];
        int acc_ri = -1;
        auto flush = [&]() {
          if (acc_ri < 0) return;
          const int rowl = (r_lo + acc_ri) * TILE_ROWS + gq;  // cluster-local row of q = 0
#pragma unroll
          for (int set = 0; set < NB; ++set) {
            const int b = set * 4 + tq;
            if (b < B) {
#pragma unroll
              for (int q = 0; q < 4; ++q) atomicAdd(part + (rowl + 8 * q) * BT + b, acc[set][q]);
            }
          }
        };
#pragma unroll 1
        for (; i < i_end; ++i) {
          if (ri != acc_ri) {
            flush();
            acc_ri = ri;
#pragma unroll
            for (int set = 0; set < NB; ++set)
#pragma unroll
              for (int q = 0; q < 4; ++q) acc[set][q] = 0.f;
          }
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
          for (int set = 0; set < NB; ++set) {  // every set (absent tokens: x' = 0): independent MMA chains
            uint4 bA = make_uint4(0u, 0u, 0u, 0u), bB = bA;  // B fragments (columns >= NCOL are zero)
            if (gq < NCOL) {
              const uint8_t* bp = xp + gi * XPG + set * XPC + tq * XTQ + gq * 32;
              bA = *reinterpret_cast<const uint4*>(bp);
              bB = *reinterpret_cast<const uint4*>(bp + 16);
            }
            constexpr uint32_t ML = 0x0f0f0f0fu, MH = 0xf0f0f0f0u;
#if PARO_G1_MERGE_NIB
            // high nibbles shifted down (q, not 16 q): both halves of the word accumulate into one
            // integer sum per (row, column) and the epilogue combines two digits, not four sums
            (void)MH;
            int D[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {  // rows gq + 16 hh (w[2 hh]) and gq + 16 hh + 8 (w[2 hh + 1])
              const uint4 r0 = w[2 * hh], r1 = w[2 * hh + 1];
              mma_u8s8(D[hh], r0.x & ML, r1.x & ML, r0.y & ML, r1.y & ML, bA.x, bA.y);
              mma_u8s8(D[hh], r0.z & ML, r1.z & ML, r0.w & ML, r1.w & ML, bA.z, bA.w);
              mma_u8s8(D[hh], (r0.x >> 4) & ML, (r1.x >> 4) & ML, (r0.y >> 4) & ML, (r1.y >> 4) & ML, bB.x, bB.y);
              mma_u8s8(D[hh], (r0.z >> 4) & ML, (r1.z >> 4) & ML, (r0.w >> 4) & ML, (r1.w >> 4) & ML, bB.z, bB.w);
            }
#else
            int Dl[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}}, Dh[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {  // rows gq + 16 hh (w[2 hh]) and gq + 16 hh + 8 (w[2 hh + 1])
              const uint4 r0 = w[2 * hh], r1 = w[2 * hh + 1];
              mma_u8s8(Dl[hh], r0.x & ML, r1.x & ML, r0.y & ML, r1.y & ML, bA.x, bA.y);
              mma_u8s8(Dl[hh], r0.z & ML, r1.z & ML, r0.w & ML, r1.w & ML, bA.z, bA.w);
              mma_u8s8(Dh[hh], r0.x & MH, r1.x & MH, r0.y & MH, r1.y & MH, bB.x, bB.y);
              mma_u8s8(Dh[hh], r0.z & MH, r1.z & MH, r0.w & MH, r1.w & MH, bB.z, bB.w);
            }
#endif
            // lane (gq, tq) holds columns 2 tq (hi) and 2 tq + 1 (lo) = token tq of the set, rows gq + 8 q
            // (tokens >= B: x' = 0 in every group, their sums never leave the CTA)
            const int b = set * 4 + tq;
            const int2 xf = xs[gi * BT + b];
            const float F = __int_as_float(xf.y);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int hh = q >> 1, e = (q & 1) * 2;
              const int zq = static_cast<int>((zw >> (4 * q)) & 15u);
#if PARO_G1_MERGE_NIB
              const int I = D[hh][e] * 256 + D[hh][e + 1] - zq * xf.x;
#else
              const int I = Dl[hh][e] * 256 + Dl[hh][e + 1] + ((Dh[hh][e] * 256 + Dh[hh][e + 1]) >> 4) - zq * xf.x;
#endif
              acc[set][q] = fmaf(Sr[q] * F, static_cast<float>(I), acc[set][q]);
            }
          }
          if (++gi == gc) {
            gi = 0;
            ++ri;
          }
        }
        flush();
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
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
    } else {
      // B > 1: 5th-generation tensor cores.  Warpgroup wg (warps 4 wg .. 4 wg + 3) takes the
      // groups gi = wg, wg + 3, .. of each batch; per group (an "item": 128 rows x 128 channels),
      // its warp j writes the A operand of row block 4 q + j into TMEM lanes 32 j .. 32 j + 31 (one
      // row per lane: the row's 16 code words, low nibbles AND 0x0F0F0F0F and high nibbles >> 4
      // AND 0x0F0F0F0F = the u8 codes of 128 channels, no conversion), one thread issues four
      // tcgen05.mma.kind::i8 (M = 128 rows, N = 2 B token digits, K = 32 each; u8 codes x s8
      // digits -> exact s32 in TMEM), and every lane reads its row back: I = 256 D_hi + D_lo - z X
      // per token, y_row += S 2^(E-14) I in registers across the CTA's groups; one shared-memory
      // atomic per (row, token) per quad.  Two A / D buffers per warpgroup: the A fill and MMA of
      // item i overlap the read-back of item i - 1.
      constexpr int NC = 2 * BT;  // MMA N: (token, digit) columns
      constexpr uint32_t IDESC = (2u << 4)                                    // D: s32
                                 | (0u << 7) | (1u << 10)                     // A: u8, B: s8
                                 | (static_cast<uint32_t>(NC >> 3) << 17)     // N >> 3
                                 | (static_cast<uint32_t>(128 >> 4) << 24);   // M >> 4
      const int wg = warp >> 2, wq = warp & 3;
      const uint32_t tbase = *tmem_slot + static_cast<uint32_t>(wg * 128);  // this warpgroup's columns
      const uint32_t lane_off = static_cast<uint32_t>(wq * 32) << 16;
      const int m = a.TPS / 4;
      const int swz = (lane >> 1) & 3;  // conflict-free row reads: chunk k ^ swz at step k
      float acc[BT];
#pragma unroll
      for (int b = 0; b < BT; ++b) acc[b] = 0.f;
      int cur_q = -1;
      // the item whose MMA is in flight
      int pend_gi = -1, pend_q = 0, pend_z = 0;
      uint32_t pend_it = 0;
      float pend_S = 0.f;
      auto flush = [&](int q) {
        const int nq = min(4, g.nrb - 4 * q);
        if (wq < nq) {
          const int row = (4 * q + wq) * TILE_ROWS + lane;  // cluster-local row
#pragma unroll
          for (int b = 0; b < BT; ++b)
            if (b < B) atomicAdd(part + row * BT + b, acc[b]);
        }
#pragma unroll
        for (int b = 0; b < BT; ++b) acc[b] = 0.f;
      };
      auto epilogue = [&]() {  // read back the pending item and accumulate
        const uint32_t buf = pend_it & 1u;
        mbar_wait_spin(&mdone[wg * 2 + buf], (pend_it >> 1) & 1u);
        tc_fence_after();
        uint32_t dv[NC];
        tmem_ld_cols<NC>(tbase + 64 + NC * buf + lane_off, dv);
        tmem_ld_wait();
        if (pend_q != cur_q) {
          if (cur_q >= 0) flush(cur_q);
          cur_q = pend_q;
        }
        // tokens >= B have x' = 0 (digits 0, sum 0): their columns add exactly 0
        const int4* xq4 = reinterpret_cast<const int4*>(xs + pend_gi * BT);
#pragma unroll
        for (int b = 0; b < BT; b += 2) {
          const int4 xf = xq4[b >> 1];  // (X, F) of tokens b and b + 1
          const int I0 = static_cast<int>(dv[2 * b]) * 256 + static_cast<int>(dv[2 * b + 1]) - pend_z * xf.x;
          const int I1 = static_cast<int>(dv[2 * b + 2]) * 256 + static_cast<int>(dv[2 * b + 3]) - pend_z * xf.z;
          acc[b] = fmaf(pend_S * __int_as_float(xf.y), static_cast<float>(I0), acc[b]);
          acc[b + 1] = fmaf(pend_S * __int_as_float(xf.w), static_cast<float>(I1), acc[b + 1]);
        }
        pend_gi = -1;
      };
#pragma unroll 1
      for (int bt = 0; bt < g.n_batches; ++bt) {
        const int q = bt / g.nch, c = bt - q * g.nch;
        const int mm = min(m, gc - c * m), nq = min(4, g.nrb - 4 * q);
        mbar_wait(&full[slot], phase);
        if (bt == 0 && tid == 0) tl_mark(s, 3);
        const uint8_t* sb = ring + static_cast<size_t>(slot) * a.slot_bytes;
#pragma unroll 1
        for (int gl = wg; gl < mm; gl += NW / 4) {
          const int gi = c * m + gl;    // CTA-local group
          const int ti = wq * mm + gl;  // tile of (row block 4 q + wq, group gi) in the batch
          const uint32_t buf = mma_it & 1u;
          uint32_t av[32];
          float Srow = 0.f;
          int zrow = 0;
          if (wq < nq) {
            const uint8_t* rp = sb + ti * TILE_CODE_BYTES + lane * 64;
            uint4 in[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) in[k] = *reinterpret_cast<const uint4*>(rp + ((k ^ swz) << 4));
            if (swz & 1) {
              uint4 t0 = in[0];
              in[0] = in[1];
              in[1] = t0;
              t0 = in[2];
              in[2] = in[3];
              in[3] = t0;
            }
            if (swz & 2) {
              uint4 t0 = in[0];
              in[0] = in[2];
              in[2] = t0;
              t0 = in[1];
              in[1] = in[3];
              in[3] = t0;
            }
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const uint32_t wv[4] = {in[t].x, in[t].y, in[t].z, in[t].w};
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                av[4 * t + j] = wv[j] & 0x0f0f0f0fu;
                av[16 + 4 * t + j] = (wv[j] >> 4) & 0x0f0f0f0fu;
              }
            }
            Srow = __half2float(*reinterpret_cast<const __half*>(sb + a.sc_off + ti * TILE_SCALE_BYTES +
                                                                 (lane & 7) * 8 + (lane >> 3) * 2));
            const uint32_t zw = *reinterpret_cast<const uint16_t*>(sb + a.z_off + ti * TILE_ZERO_BYTES + (lane & 7) * 2);
            zrow = static_cast<int>((zw >> (4 * (lane >> 3))) & 15u);
          } else {
#pragma unroll
            for (int k = 0; k < 32; ++k) av[k] = 0u;
          }
          tmem_st32(tbase + 32 * buf + lane_off, av);
          tmem_st_wait();
          tc_fence_before();
          // A complete; every warp has read back the item that last used these buffers
          named_bar_sync(5 + wg, 128);
          if (wq == 0 && lane == 0) {
            tc_fence_after();
            const uint64_t bd = smem_desc_sw128(xp + gi * XPG);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_i8_ts(tbase + 64 + NC * buf, tbase + 32 * buf + 8 * kk, bd + 2 * kk, IDESC, kk > 0 ? 1u : 0u);
            mma_commit(&mdone[wg * 2 + buf]);
          }
          if (pend_gi >= 0) epilogue();  // the previous item, while this one multiplies
          pend_gi = gi;
          pend_q = q;
          pend_S = Srow;
          pend_z = zrow;
          pend_it = mma_it++;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);  // the batch's data is in TMEM / registers
        if (++slot == a.S) {
          slot = 0;
          phase ^= 1;
        }
      }
      if (pend_gi >= 0) epilogue();
      if (cur_q >= 0) flush(cur_q);
    }

    // ---------------------------------------------------------- reduction + epilogue (a8)
    named_bar_sync(1, NW * 32);
    if (tid == 0) tl_mark(s, 4);
    if (s == 0 && CL > 1) cluster_wait();  // every CTA of the cluster is running: DSMEM is legal
    if (BT > 1 && g.active) {
      // four tokens per st.async (16 B), owner by owner (no per-element division)
      constexpr int Q4 = BT >= 4 ? BT / 4 : 1;  // (BT = 1 never takes this branch)
#pragma unroll 1
      for (int c = 0, r0 = 0; c < CL && r0 < g.R; ++c, r0 += g.RR) {
        const int rows = min(g.RR, g.R - r0);
#pragma unroll 1
        for (int idx = tid; idx < rows * Q4; idx += NW * 32) {
          const int rl = idx / Q4, q = idx & (Q4 - 1);
          const uint4 v = *reinterpret_cast<const uint4*>(part + (r0 + rl) * BT + 4 * q);
          float* dst = recv + (crank * S.RRmax + rl) * BT + 4 * q;
          if (c == crank)
            *reinterpret_cast<uint4*>(dst) = v;
          else
            st_async_v4(mapa(smem_u32(dst), static_cast<uint32_t>(c)), v,
                        mapa(smem_u32(rbar), static_cast<uint32_t>(c)));
        }
      }
    } else if (g.active) {
      for (int idx = tid; idx < g.R * BT; idx += NW * 32) {
        const int r = idx / BT, b = idx - r * BT;
        float sum;
        if (BT == 1 && !S.atom) {
          float s4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
          for (int w = 0; w < NW; ++w) s4[w & 3] += part[static_cast<size_t>(w) * S.R_max + r];
          sum = (s4[0] + s4[1]) + (s4[2] + s4[3]);  // fixed order
        } else {
          sum = part[idx];
        }
        const int owner = r / g.RR;
        float* dst = recv + (crank * S.RRmax + (r - owner * g.RR)) * BT + b;
        if (owner == crank)
          *dst = sum;
        else
          st_async_b32(mapa(smem_u32(dst), static_cast<uint32_t>(owner)), __float_as_uint(sum),
                       mapa(smem_u32(rbar), static_cast<uint32_t>(owner)));
      }
    }
    named_bar_sync(1, NW * 32);           // my own partials are in recv
    if (g.active && CL > 1) mbar_wait(rbar, s & 1);  // and those of the other CTAs of the cluster
    if (tid == 0) tl_mark(s, 5);
    if (g.active) {
      for (int idx = tid; idx < g.my_n * BT; idx += NW * 32) {
        const int rl = idx / BT, b = idx - rl * BT;
        if (b >= B) continue;
        float v = 0.f;
        for (int c = 0; c < CL; ++c) v += recv[(c * S.RRmax + rl) * BT + b];  // fixed order
        const int64_t n = static_cast<int64_t>(g.rb0) * TILE_ROWS + g.my_lo + rl;
        if (n < d.N) {
          if (d.bias) v += __ldg(d.bias + n);
          const int64_t o = static_cast<int64_t>(b) * d.N + n;
          if (a.y_dtype == 0)
            static_cast<__half*>(d.y)[o] = __float2half_rn(v);
          else if (a.y_dtype == 1)
            static_cast<__nv_bfloat16*>(d.y)[o] = __float2bfloat16_rn(v);
          else
            static_cast<float*>(d.y)[o] = v;
        }
      }
    }
    if (tid == 0) tl_mark(s, 6);
    if (s + 1 < n_st) {
      named_bar_sync(1, NW * 32);  // every store (and every read of recv) of this stage is done
      if (tid == 0) {
        if (CL > 1)  // the next stage's cluster partials may land once the barrier below completes
          mbar_arrive_expect_tx(rbar, static_cast<uint32_t>((CL - 1) * sgeo[s + 1].my_n * BT * 4));
      }
      arrive_grid();
    }
  }
  // the next launch on this workspace uses the next epoch (it reads the word only after this
  // grid completed: PDL wait or stream order)
  if (n_st > 1 && blockIdx.x == 0 && tid == 0) st_relaxed_gpu(gb.epoch, (ep >> 6) + 1);
  if constexpr (UM) {  // every warpgroup waited for its last MMA
    tc_fence_before();
    named_bar_sync(1, NW * 32);
    if (warp == 2) tmem_dealloc(*tmem_slot, 512);
  }
}

// Activation transform of stage 0 for B > 1 (a4, a5), once per (linear, group, set of four
// tokens) for the whole launch: one warp each.
struct Gemv1XformArgs {
  Gemv1Stage st;
  int B, x_bf16, rotate, pdl;
};

template <int BT, bool UM>
__global__ void __launch_bounds__(128) paro_gemv1_xform_kernel(const __grid_constant__ Gemv1XformArgs a) {
  __shared__ __align__(16) float scr_all[4][128];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (a.pdl) pdl_launch_dependents();
  const int task = blockIdx.x * 4 + warp;
  if (task >= a.st.n_lin * a.st.G * BT) return;
  g1_xform_task<BT, UM>(a.st, task, a.B, a.x_bf16, a.rotate, scr_all[warp], lane, a.pdl != 0);
}

// ============================================================================ host side
// Plan overrides for experiments exist only in builds with -DPARO_DEBUG_KNOBS=1 (never in
// the shipped library: a stray environment variable must not change what a call computes).
static int g1_env(const char* name, int dflt) {
#if PARO_DEBUG_KNOBS
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
#else
  (void)name;
  return dflt;
#endif
}

static inline uint32_t g1_align(uint32_t v, uint32_t al) { return (v + al - 1) / al * al; }

bool gemv1_enabled() { return g1_env("PARO_GEMV1", 1) != 0; }

size_t gemv1_xq_bytes(int B, int64_t K) {
  if (B <= 1) return 0;
  const int BT = B <= 4 ? 4 : B <= 8 ? 8 : 16;
  const size_t G = static_cast<size_t>(K / 128);
  // per group GEMV1_XQ_GROUP_BYTES (4 KB) of x' digits (BT / 4 KB used), then the
  // per-(group, token) sums / scales at G * 4096
  return (G * GEMV1_XQ_GROUP_BYTES + G * BT * 8 + 255) / 256 * 256;
}

cudaError_t launch_gemv1_xform(const Gemv1Config& c, cudaStream_t st) {
  Gemv1XformArgs x{};
  x.st = c.a.st[0];
  x.B = c.a.B;
  x.x_bf16 = c.a.x_bf16;
  x.rotate = c.a.rotate;
  x.pdl = c.a.pdl;
  const int tasks = x.st.n_lin * x.st.G * c.BT;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((tasks + 3) / 4);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute at;
  at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at.val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = &at;
  cfg.numAttrs = x.pdl ? 1 : 0;
  switch (c.BT) {
    case 4: return c.a.umma ? cudaLaunchKernelEx(&cfg, paro_gemv1_xform_kernel<4, true>, x)
                            : cudaLaunchKernelEx(&cfg, paro_gemv1_xform_kernel<4, false>, x);
    case 8: return c.a.umma ? cudaLaunchKernelEx(&cfg, paro_gemv1_xform_kernel<8, true>, x)
                            : cudaLaunchKernelEx(&cfg, paro_gemv1_xform_kernel<8, false>, x);
    case 16: return c.a.umma ? cudaLaunchKernelEx(&cfg, paro_gemv1_xform_kernel<16, true>, x)
                             : cudaLaunchKernelEx(&cfg, paro_gemv1_xform_kernel<16, false>, x);
    default: return cudaErrorInvalidConfiguration;
  }
}

template <int BT, int MS, bool UM>
static const void* g1_kernel() {
  return reinterpret_cast<const void*>(&paro_gemv1_kernel<g1_nw(BT, UM, MS > 1), BT, MS, UM>);
}
template <int MS, bool UM>
static const void* g1_kernel_ms(int BT) {
  return BT == 1 ? g1_kernel<1, MS, false>() : BT == 4 ? g1_kernel<4, MS, UM>() : BT == 8 ? g1_kernel<8, MS, UM>()
                                                                                            : g1_kernel<16, MS, UM>();
}
static const void* g1_kernel_bt(int BT, bool chain, bool um) {
  if (chain) return um ? g1_kernel_ms<CHAIN_MAX_STAGES, true>(BT) : g1_kernel_ms<CHAIN_MAX_STAGES, false>(BT);
  return um ? g1_kernel_ms<1, true>(BT) : g1_kernel_ms<1, false>(BT);
}

// clusters of CL (BT-token instance) that fit in one wave, from the occupancy API (cached per
// device)
static int g1_active_clusters_compute(const void* k, int CL, int threads, int budget) {
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
static int g1_active_clusters(int BT, bool chain, bool um, int CL, int threads, int budget) {
  return cached_device_int(g1_kernel_bt(BT, chain, um), CL, threads, budget, g1_active_clusters_compute);
}

bool plan_gemv1_chain(int B, int n_stages, const int* n_lin, const int64_t (*Ns)[GEMV_MAX_LIN], const int64_t* Ks,
                      int rotate, int tcgen05, Gemv1Config* cfg, const char** why) {
  if (B < 1 || B > GEMV1_MAX_B) {
    *why = "1..16 tokens per decode launch";
    return false;
  }
  if (n_stages < 1 || n_stages > CHAIN_MAX_STAGES) {
    *why = "1..16 stages per decode launch";
    return false;
  }
  const bool chain = n_stages > 1;
  const int BT = B == 1 ? 1 : B <= 4 ? 4 : B <= 8 ? 8 : 16;
  const bool um = BT > 1 && tcgen05;
  const int NSET = (BT + 3) / 4;
  int Gmin = 1 << 30;
  double wbytes = 0;
  for (int s = 0; s < n_stages; ++s) {
    if (n_lin[s] < 1 || n_lin[s] > GEMV_MAX_LIN) {
      *why = "1..4 linears per decode stage";
      return false;
    }
    const int G = static_cast<int>(Ks[s] / 128);
    if (G < 1) {
      *why = "K must be a positive multiple of 128";
      return false;
    }
    Gmin = std::min(Gmin, G);
    for (int i = 0; i < n_lin[s]; ++i) wbytes += static_cast<double>(Ns[s][i]) * Ks[s] * 0.52;
  }
  Gemv1Config c{};
  Gemv1Args& a = c.a;
  // Cluster size = how many ways a row block's groups are split (G / CL groups transformed per
  // CTA).  The rotations are shared-memory bound (8 accesses per pair-update, all warps at once),
  // so fewer groups per CTA shorten the transform; but clusters of 2 / 4 / 8 fill only 148 / 132
  // / 120 SMs (occupancy API), which slows the weight stream.  Measured for single launches
  // (tools/time_groups.py, tools/time_70b.py): short streams (< 20 MB) at K = 4096 prefer 4, long
  // ones 2; K >= 8192 prefers 8 (one transform round) unless the stream is very long and G small
  // (70B gate+up: 2).  A chain shares one cluster size over its stages: 4.
  int CL;
  if (chain) {
    CL = 4;
  } else {
    const int G = static_cast<int>(Ks[0] / 128);
    if (G >= 64)
      CL = (wbytes < 64e6 || G >= 128) ? 8 : 2;
    else
      CL = wbytes < 20e6 ? 4 : 2;
  }
  CL = g1_env(chain ? "PARO_G1_CHAIN_CL" : "PARO_G1_CL", CL);
  if (CL != 1 && CL != 2 && CL != 4 && CL != 8) CL = 2;
  while (CL > 1 && CL > Gmin) CL /= 2;
  const int NW = g1_nw(BT, um, chain);
  const int threads = (NW + 1) * 32;
  c.NW = NW;
  // B > 1 single launches: 3 KB of the SM's shared memory stay free for a co-resident pre-kernel CTA
  const int budget = device_smem_optin() - 1024 - ((PARO_G1_COXFORM && BT > 1 && !chain) ? 3072 : 0);
  int ncl_max = g1_active_clusters(BT, chain, um, CL, threads, budget);
  ncl_max = std::min(ncl_max, std::max(1, g1_env("PARO_G1_MAXCL", 1 << 20)));
  int grid = 0, rmax_all = 0, rrmax_all = 0, gcm = 0, part_words = 0;
  int64_t cta_tiles = 0;  // tiles of the busiest CTA over the whole chain
  for (int s = 0; s < n_stages; ++s) {
    Gemv1Stage& S = a.st[s];
    const int n = n_lin[s];
    const int G = static_cast<int>(Ks[s] / 128);
    // clusters over linears in proportion to their row blocks (>= 1 each, <= row blocks)
    int64_t NB[GEMV_MAX_LIN], NBsum = 0;
    for (int i = 0; i < n; ++i) {
      NB[i] = (Ns[s][i] + TILE_ROWS - 1) / TILE_ROWS;
      NBsum += NB[i];
    }
    int ncl = static_cast<int>(std::min<int64_t>(ncl_max, NBsum));
    if (ncl < n) ncl = n;
    int cls[GEMV_MAX_LIN], used = 0, big = 0;
    for (int i = 0; i < n; ++i) {
      cls[i] = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(NB[i], ncl * NB[i] / NBsum)));
      used += cls[i];
      if (NB[i] > NB[big]) big = i;
    }
    cls[big] = static_cast<int>(std::min<int64_t>(NB[big], cls[big] + std::max(0, ncl - used)));
    int begin = 0, rmax = 0;
    for (int i = 0; i < n; ++i) {
      Gemv1Linear& d = S.lin[i];
      d.N = static_cast<int>(Ns[s][i]);
      d.cta_begin = begin;
      d.rb_base = static_cast<int>(NB[i] / cls[i]);
      d.rb_extra = static_cast<int>(NB[i] % cls[i]);
      rmax = std::max(rmax, (d.rb_base + (d.rb_extra ? 1 : 0)) * TILE_ROWS);
      begin += cls[i] * CL;
    }
    S.n_lin = n;
    S.K = static_cast<int>(Ks[s]);
    S.G = G;
    S.n_cta = begin;
    S.R_max = rmax;
    S.RRmax = (rmax + CL - 1) / CL;
    // B = 1: per-warp row partials summed in a fixed order (deterministic) while they fit in
    // 48 KB; clusters with more rows (e.g. 70B gate+up: 3840 rows) add with shared atomics
    S.atom = BT == 1 && (static_cast<int64_t>(NW) * rmax * 4 > (g1_env("PARO_G1_ATOM_KB", 48) << 10));
    S.xq_in_kernel = (BT > 1 && s > 0) ? 1 : 0;
    grid = std::max(grid, begin);
    rmax_all = std::max(rmax_all, rmax);
    rrmax_all = std::max(rrmax_all, S.RRmax);
    gcm = std::max(gcm, (G + CL - 1) / CL);
    part_words = std::max(part_words, (BT == 1 && !S.atom ? NW : BT) * rmax);
    cta_tiles += static_cast<int64_t>(rmax / TILE_ROWS) * ((G + CL - 1) / CL);
  }
  c.grid = grid;
  c.CL = CL;
  c.BT = BT;
  a.B = B;
  a.umma = um ? 1 : 0;
  a.n_stages = n_stages;
  a.rotate = rotate;
  a.pre_stages = std::max(0, g1_env("PARO_G1_PRE", 2));
  a.params_first = g1_env("PARO_G1_PF", 1);
  a.l2_batches = g1_env("PARO_G1_L2B", 4);
  a.xfirst = g1_env("PARO_G1_XFIRST", 1);
  a.nobar = g1_env("PARO_G1_NOBAR", 0);
  uint32_t off = 0;
  a.off_xp = off;
  off += g1_align(static_cast<uint32_t>(gcm) * NSET * 4 * (BT == 1 ? 2 : 8) * 32, 128);
  off += 128;  // 32 zero bytes (lanes of unused MMA columns) just below xs
  a.off_xs = off;
  off += g1_align(static_cast<uint32_t>(gcm) * BT * 8, 128);
  a.off_part = off;
  off += g1_align(static_cast<uint32_t>(part_words) * 4, 128);
  a.off_scr = off;
  if (BT == 1 || chain) off += NW * 512;  // per-warp 128-channel scratch (B > 1: later stages' transform tasks)
  a.off_recv = off;
  off += g1_align(static_cast<uint32_t>(CL) * rrmax_all * BT * 4, 128);
  a.off_bar = off;
  off += 64 * 16 + 64;  // <= 128 mbarriers (ring full / empty <= 2 x 56, rbar, xbar, 8 x mdone) + the TMEM base
  a.off_ring = g1_align(off, 1024);
  // B > 1 aligns the dynamic shared-memory base to 1024 B at run time (UMMA swizzle): reserve the slack
  const int64_t avail = static_cast<int64_t>(budget) - (um ? 1024 : 0) - a.off_ring;
  // batch size: the TPS that keeps the most tiles in flight (ring depth x batch size, capped by
  // the CTA's tiles), >= 2 batches in the ring unless one holds everything; measured: the
  // HBM stream is bound by the bytes a CTA has in flight (LLaMA-3-8B gate+up at 15 warps: 30 tiles
  // x 2 batches 15.7 us, 28 x 3 14.0 us)
  auto slot_of = [&](int tps) {
    const uint32_t sc = static_cast<uint32_t>(tps) * TILE_CODE_BYTES;
    return g1_align(sc + static_cast<uint32_t>(tps) * (TILE_SCALE_BYTES + TILE_ZERO_BYTES), 128);
  };
  auto stages_of = [&](int tps) {
    const int64_t need = (cta_tiles + tps - 1) / tps + n_stages;
    return std::min<int64_t>(std::min<int64_t>(need, 56), avail / slot_of(tps));
  };
  int TPS = g1_env("PARO_G1_TPS", 0);
  if (TPS <= 0 || TPS > 64) {
    int best = 0;
    int64_t best_in = -1;
    const int step = um ? 4 : 2;
    for (int tps = (2 * NW) / step * step; tps >= 12; tps -= step) {
      const int64_t S_ = stages_of(tps), nbat = (cta_tiles + tps - 1) / tps;
      if (S_ < std::min<int64_t>(2, nbat)) continue;
      const int64_t in = std::min(S_, nbat) * tps;
      if (in > best_in) {
        best_in = in;
        best = tps;
      }
    }
    TPS = best ? best : 8;
  }
  a.TPS = TPS;
  a.sc_off = static_cast<uint32_t>(TPS) * TILE_CODE_BYTES;
  a.z_off = a.sc_off + static_cast<uint32_t>(TPS) * TILE_SCALE_BYTES;
  a.slot_bytes = slot_of(TPS);
  const int S = static_cast<int>(stages_of(TPS));
  if (S < 1) {
    *why = "decode shared-memory plan does not fit";
    return false;
  }
  a.S = S;
  a.smem_total = a.off_ring + static_cast<uint32_t>(S) * a.slot_bytes + (um ? 1024 : 0);
  if (g1_env("PARO_PLAN_DEBUG", 0))
    fprintf(stderr, "[paro gemv1 plan] B=%d BT=%d stages=%d grid=%d CL=%d NW=%d TPS=%d S=%d R_max=%d smem=%u\n", B, BT,
            n_stages, c.grid, CL, NW, TPS, S, rmax_all, a.smem_total);
  *cfg = c;
  return true;
}

bool plan_gemv1(int B, int n_lin, const int64_t* Ns, int64_t K, int rotate, int tcgen05, Gemv1Config* cfg,
                const char** why) {
  int64_t ns[1][GEMV_MAX_LIN] = {};
  for (int i = 0; i < n_lin && i < GEMV_MAX_LIN; ++i) ns[0][i] = Ns[i];
  return plan_gemv1_chain(B, 1, &n_lin, ns, &K, rotate, tcgen05, cfg, why);
}

template <int BT, int MS, bool UM>
static cudaError_t g1_launch(const Gemv1Config& c, cudaLaunchConfig_t* cfg) {
  auto kern = paro_gemv1_kernel<g1_nw(BT, UM, MS > 1), BT, MS, UM>;
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), static_cast<int>(c.a.smem_total));
  if (e != cudaSuccess) return e;
  if constexpr (MS == CHAIN_MAX_STAGES) {
    return cudaLaunchKernelEx(cfg, kern, c.a);
  } else {
    // one-stage argument block (smaller kernel parameters)
    Gemv1ArgsT<MS> a1;
    static_assert(sizeof(Gemv1ArgsT<MS>) <= sizeof(Gemv1Args), "");
    std::memcpy(static_cast<void*>(&a1), static_cast<const void*>(&c.a), sizeof(a1));
    return cudaLaunchKernelEx(cfg, kern, a1);
  }
}

cudaError_t launch_gemv1(const Gemv1Config& c, cudaStream_t st) {
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
  const bool chain = c.a.n_stages > 1;
  const bool um = c.a.umma != 0;
#define G1_L(BT_)                                                                                              \
  (chain ? (um ? g1_launch<BT_, CHAIN_MAX_STAGES, true>(c, &cfg) : g1_launch<BT_, CHAIN_MAX_STAGES, false>(c, &cfg)) \
         : (um ? g1_launch<BT_, 1, true>(c, &cfg) : g1_launch<BT_, 1, false>(c, &cfg)))
  switch (c.BT) {
    case 1: return chain ? g1_launch<1, CHAIN_MAX_STAGES, false>(c, &cfg) : g1_launch<1, 1, false>(c, &cfg);
    case 4: return G1_L(4);
    case 8: return G1_L(8);
    case 16: return G1_L(16);
    default: return cudaErrorInvalidConfiguration;
  }
#undef G1_L
}

}  // namespace paro
