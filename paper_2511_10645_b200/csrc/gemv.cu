// gemv.cu -- decode path (B <= 8 tokens per launch): scale + L Givens layers fused
// into the activation staging, then the group-wise INT4 dequant GEMV on the warp-level
// tensor cores.
//
// SURVEY.md 8(a) rows a4 (stage + scale), a5 (L rotations, Eq. 5 in column form),
// a6 (dequant GEMV), a8 (epilogue).  One kernel, launched as clusters of CL CTAs
// (1-2 CTAs per SM, one wave).  A cluster owns a run of 32-row blocks of one linear;
// the tiles (32 rows x one 128-group, tile_layout.cuh) of that run are split evenly and
// contiguously over its CL CTAs (split-K at tile granularity, so every CTA streams the
// same number of bytes whatever N and K are).
//
//  * producer warp: bulk-copies (cp.async.bulk, TMA engine) first the rotation
//    parameters and the activations this CTA transforms, then its contiguous tile range
//    (codes / scales / zeros are three contiguous ranges) through a ring of
//    shared-memory stages (TPS tiles each), completion tracked by mbarriers.
//  * compute warps, phase 1 (transform; PAPER.md:195-209's token / group / pair
//    parallelism): the CL CTAs of a cluster split the K/128 groups; a warp owns a
//    group, stages it in shared memory, scales by s and applies the L independent
//    rotations (2 pairs per lane per rotation, sync-free inside a rotation, __syncwarp
//    between rotations; the pack-time schedule makes every gather / scatter
//    bank-conflict free).  The fp16 x' of the group -- laid out as mma.sync B fragments
//    -- and its per-token sum go to every CTA of the cluster with st.async (DSMEM),
//    completion counted in bytes on the receiver's mbarrier.  x' never goes to HBM.
//  * compute warps, phase 2 (GEMV): warp w takes tiles w, w + NW, ... of each stage.
//    Lane (g, t) loads 16 code bytes of rows g, g + 8, g + 16, g + 24 (four LDS.128); one
//    AND mask per 32-bit word turns 2 nibbles into an fp16 A-fragment register: a nibble
//    q in bits [0,4) of a half IS the subnormal q * 2^-24 (bits [4,8): 16q * 2^-24), which
//    the tensor cores multiply exactly.  Sixteen mma.sync.m16n8k16 per tile (two 16-row
//    blocks, four per power-of-two scale each, four independent accumulator chains) give
//    sum_k q[n,k] x'[k, b] for the 32 rows x 8 token columns, sharing one set of B
//    fragments;
//    the epilogue applies y += S * (sum q x' - z * sum x') per (row, group, token).
//    Row partials of a warp go to shared memory when its row block changes; warps are
//    summed in a fixed order, and the CTA holding the first tile of a row block adds
//    the partials of the (at most CL - 1) later CTAs that share it, pushed to it with
//    st.async -- deterministic, no atomics.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "paro_internal.h"
#include "ptx.cuh"
#include "tile_layout.cuh"

namespace paro {

constexpr int GRP = 128;
constexpr float TWO_P24 = 16777216.0f;  // 2^24
constexpr int TL_EVENTS = 12;           // debug timeline: events per CTA
constexpr uint32_t TILE_BYTES = TILE_CODE_BYTES + TILE_SCALE_BYTES + TILE_ZERO_BYTES;


__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#ifndef PARO_ENABLE_DEBUG
#define PARO_ENABLE_DEBUG 0  // 1: per-launch timeline / cycle counters (flag 0x100; tools/timeline.py). Off: ~5% faster
#endif
#if PARO_ENABLE_DEBUG
__device__ unsigned long long g_paro_timeline[1024 * TL_EVENTS];
__device__ unsigned long long g_paro_prof[1024 * 16 * 8];  // debug: per (CTA, warp) cycle counters
#else
__device__ unsigned long long* const g_paro_timeline = nullptr;
__device__ unsigned long long* const g_paro_prof = nullptr;
#endif
#define PARO_DBG(a) (PARO_ENABLE_DEBUG && (a).debug)
#define PARO_TL(a, ev)                                                                            \
  do {                                                                                            \
    if (PARO_DBG(a) && blockIdx.x < 1024) g_paro_timeline[blockIdx.x * TL_EVENTS + (ev)] = gtimer(); \
  } while (0)

__device__ __forceinline__ uint32_t pack_half2(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ float load_act(const void* x, int bf16, int64_t i) {
  if (bf16) return __bfloat162float(static_cast<const __nv_bfloat16*>(x)[i]);
  return __half2float(static_cast<const __half*>(x)[i]);
}

__device__ __forceinline__ void store_out(void* y, int dt, int64_t i, float v) {
  if (dt == 0)
    static_cast<__half*>(y)[i] = __float2half_rn(v);
  else if (dt == 1)
    static_cast<__nv_bfloat16*>(y)[i] = __float2bfloat16_rn(v);
  else
    static_cast<float*>(y)[i] = v;
}

__device__ __forceinline__ float half2_sum(uint32_t w) {
  const float2 f = __half22float2(*reinterpret_cast<__half2*>(&w));
  return f.x + f.y;
}

// first cluster-local tile of cluster CTA k (tiles split evenly and contiguously); CL is a
// power of two, lcl = log2(CL): shifts, no integer division
__device__ __forceinline__ int cta_tile_start(int k, int nt, int lcl) { return (k * nt) >> lcl; }
// the CTA whose (non-empty) range holds cluster-local tile x
__device__ __forceinline__ int cta_of_tile(int x, int nt, int lcl) {
  int k = 0;
  for (int c = 1; c < (1 << lcl); ++c)
    if (cta_tile_start(c, nt, lcl) <= x) k = c;
  return k;
}

// BT: token tile (1, 2, 4, 8; a.B <= BT live tokens), compile-time so the per-token loops
// of the transform unroll (a runtime token loop costs ~3.5x in the rotation latency).
// MAXT: 288 (<= 8 compute warps, 2 CTAs / SM), 512 (<= 15) or 640 (<= 19).  Registers are
// allocated per SM sub-partition (16K each, warps round-robin), so 16 warps get up to 128
// registers per thread while 17..20 warps get 96.
// IM: integer tensor-core variant for BT <= 2 (see the header comment, "IMMA path").
template <int BT, int MAXT, bool IM>
__global__ void __launch_bounds__(MAXT, MAXT <= 288 ? 2 : 1) paro_gemv_kernel(const GemvArgs a) {
  static_assert(!IM || BT <= 2, "the IMMA path holds at most two tokens per launch");
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int NW = a.NW;
  const bool is_producer = warp == NW;
  // which linear this CTA serves (CTA ranges are whole clusters)
  int li = 0;
  while (li + 1 < a.n_lin && static_cast<int>(blockIdx.x) >= a.lin[li + 1].cta_begin) ++li;
  const GemvLinear& d = a.lin[li];
  const int K = a.K, G = a.G, L = d.L, B = a.B;
  const int CL = static_cast<int>(cluster_nctarank());
  const int crank = static_cast<int>(cluster_ctarank());
  const int lcl = __ffs(CL) - 1;  // CL is 1, 2, 4 or 8
  // this cluster's row blocks and this CTA's tile range [tA, tE) (cluster-local indices)
  const int cl = (static_cast<int>(blockIdx.x) - d.cta_begin) / CL;
  const int nrb_c = d.rb_base + (cl < d.rb_extra ? 1 : 0);
  const int rbc0 = cl * d.rb_base + min(cl, d.rb_extra);
  const int nt = nrb_c * G;
  const int tA = cta_tile_start(crank, nt, lcl), tE = cta_tile_start(crank + 1, nt, lcl);
  const int n_my = tE - tA;
  const int TPS = a.TPS;
  const int n_stages = (n_my + TPS - 1) / TPS;
  const int rho_first = n_my > 0 ? tA / G : 0;  // cluster-local row block of my first tile
  const int n_rho = n_my > 0 ? (tE - 1) / G - rho_first + 1 : 0;
  const bool own_first = n_my > 0 && rho_first * G >= tA;                // its first tile is mine
  const bool own_last = n_my > 0 && (rho_first + n_rho - 1) * G >= tA;  // likewise for my last block
  // later CTAs of the cluster that share my last row block (they push their partials)
  int last_cta = crank;
  if (own_last && (rho_first + n_rho) * G > tE) last_cta = cta_of_tile((rho_first + n_rho) * G - 1, nt, lcl);

  uint8_t* ufr = smem + a.off_u;                                  // x' fragments [G][4][BT][4][4] u32
  float* xsum = reinterpret_cast<float*>(smem + a.off_xs);        // sum of x' per (group, token) [G][8]
  float* part = reinterpret_cast<float*>(smem + a.off_part);      // [NW][R_max][32][BT]
  float* recv = reinterpret_cast<float*>(smem + a.off_recv);      // [CL-1][32][BT]
  uint8_t* ring = smem + a.off_ring;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.off_bar);
  uint64_t* empty = full + a.S;
  uint64_t* xpbar = empty + a.S;  // x' of all K landed (DSMEM st.async from the cluster)
  uint64_t* rbar = xpbar + 1;    // partials of my last row block from later CTAs landed

  // groups whose transform this CTA computes
  const int g_per = (G + CL - 1) / CL;
  const int g0 = min(G, crank * g_per);
  const int g1 = min(G, g0 + g_per);
  const int L_eff = a.rotate ? L : 0;

  if (threadIdx.x == 0) {
    PARO_TL(a, 0);
    for (int i = 0; i < a.S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NW);
    }
    mbar_init(xpbar, 1);
    mbar_init(rbar, 1);
    if (CL > 1) mbar_arrive_expect_tx(xpbar, static_cast<uint32_t>(BT) * (K * 2 + G * (IM ? 8 : 4)));
    uint32_t rbytes = 0;
    for (int c = crank + 1; c <= last_cta; ++c)
      if (cta_tile_start(c + 1, nt, lcl) > cta_tile_start(c, nt, lcl)) rbytes += TILE_ROWS * B * 4;
    if (rbytes) mbar_arrive_expect_tx(rbar, rbytes);
    fence_mbar_init();
  }
  // Barriers are initialised; arrive on the cluster barrier (release) now but wait on it
  // only right before the first DSMEM access, so the copies below are not held back by
  // the launch skew between the CTAs of a cluster.
  __syncthreads();
  if (CL > 1) cluster_arrive();
  if (a.pdl) pdl_launch_dependents();

  // ------------------------------------------------------------ producer warp
  if (is_producer) {
    const uint64_t pol = l2_evict_first_policy();
    const int64_t tile0 = static_cast<int64_t>(rbc0) * G + tA;  // my first tile (global index)
    auto issue = [&](int st, int slot) {
      const int64_t T = tile0 + static_cast<int64_t>(st) * TPS;
      const uint32_t nts = static_cast<uint32_t>(min(TPS, n_my - st * TPS));
      uint8_t* dst = ring + static_cast<size_t>(slot) * a.slot_bytes;
      mbar_arrive_expect_tx(&full[slot], nts * TILE_BYTES);
      bulk_g2s(dst, d.codes + T * TILE_CODE_BYTES, nts * TILE_CODE_BYTES, &full[slot], pol);
      bulk_g2s(dst + a.sc_off, d.scales + T * TILE_SCALE_BYTES, nts * TILE_SCALE_BYTES, &full[slot], pol);
      bulk_g2s(dst + a.z_off, d.zeros + T * TILE_ZERO_BYTES, nts * TILE_ZERO_BYTES, &full[slot], pol);
    };
    const int first = min(a.S, n_stages);
    // Request order: the transform warps' parameter and activation loads first (they are on
    // the critical path and would otherwise queue behind the whole GPU's ring fill), then the
    // weight ring.  Under PDL a couple of stages go out before waiting for them: the weights
    // are never written by the previous kernel (PARO_LINEAR_PDL's contract), and its tail
    // leaves HBM idle.
    const int early = a.pdl ? min(a.early_stages, first) : 0;
    // when the ring will be refilled, the first stage lands before the rest is requested
    const int stag = (a.stagger > 0 && n_stages > a.S) ? max(early, min(a.stagger, first)) : -1;
    bool synced = !a.xfirst;
    for (int st = 0; st < n_stages; ++st) {  // one issue site (small code: instruction cache)
      if (!synced && st >= early) {
        named_bar_sync(2, (NW + 1) * 32);  // the transform warps have issued their loads
        synced = true;
      }
      if (st == stag) mbar_wait(&full[0], 0);
      const int slot = st % a.S;
      if (st >= a.S) mbar_wait(&empty[slot], ((st / a.S) & 1) ^ 1);  // stage st - S consumed by every warp
      if (lane == 0) issue(st, slot);
    }
    if (!synced) named_bar_sync(2, (NW + 1) * 32);
    __syncwarp();
    if (CL > 1) cluster_wait();
    return;
  }

  // ------------------------------------------------------------ phase 1: activation transform
  {
    float* scr = reinterpret_cast<float*>(smem + a.off_scr) + warp * (a.scr_groups * BT * 132);
    const uint32_t scr_a = smem_u32(scr);
    const uint32_t u_addr = smem_u32(ufr), s_addr = smem_u32(xsum), bar_addr = smem_u32(xpbar);
    // output: lane (i4, t4, hf) writes B-fragment registers 4*i4 + 2*hf, +1 of fragment lane t4
    // (MMA m = 2*i4 + hf: channels (16m + 2t4, +1) and (16m + 2t4 + 8, +9))
    const int i4 = lane >> 3, t4 = (lane >> 1) & 3, hf = lane & 1;
    const int k0 = 16 * (2 * i4 + hf) + 2 * t4;
    bool cwaited = false;
    unsigned long long q0 = 0, q_par = 0, q_rot = 0, q_out = 0;

    // rotation parameters + s of one group -> registers (records [group][t][32 lanes]:
    // (cos0, sin0, cos1, sin1) and (i0, j0, i1, j1) of slots lane, lane + 32)
    auto load_params = [&](int gam, float4 (&cs)[8], uint32_t (&ix)[8], float4& sv) {
      const int64_t rec = static_cast<int64_t>(gam) * L * 32 + lane;
#pragma unroll
      for (int t = 0; t < 8; ++t)
        if (t < L_eff) {
          cs[t] = __ldg(reinterpret_cast<const float4*>(d.rot_cs) + rec + t * 32);
          ix[t] = __ldg(reinterpret_cast<const uint32_t*>(d.rot_idx) + rec + t * 32);
        }
      sv = a.rotate ? __ldg(reinterpret_cast<const float4*>(d.svec + gam * GRP) + lane) : make_float4(1.f, 1.f, 1.f, 1.f);
    };
    // x' = R_L ... R_1 diag(s) x of NG groups (in lockstep: independent dependency chains)
    // for the BT tokens, written as B fragments (+ per-token sums) into every CTA of the cluster
    // xr: activations (channels 4*lane .. 4*lane + 3 of each group, straight from L2)
    auto process = [&](auto ngc, const int* gams, const float4 (*csr)[8], const uint32_t (*ixr)[8],
                       const float4* sv, const uint2 (*xr)[BT]) {
      constexpr int NG = decltype(ngc)::value;
      if (PARO_DBG(a)) q0 = clock64();
#pragma unroll
      for (int q = 0; q < NG; ++q) {
#pragma unroll
        for (int b = 0; b < BT; ++b) {  // a4: diag(s) x, lane = channels 4*lane .. 4*lane + 3
          const uint2 xv = xr[q][b];
          float2 f01, f23;
          if (a.x_bf16) {
            f01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xv.x));
            f23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xv.y));
          } else {
            f01 = __half22float2(*reinterpret_cast<const __half2*>(&xv.x));
            f23 = __half22float2(*reinterpret_cast<const __half2*>(&xv.y));
          }
          *reinterpret_cast<float4*>(scr + (q * BT + b) * 132 + 4 * lane) =
              make_float4(f01.x * sv[q].x, f01.y * sv[q].y, f23.x * sv[q].z, f23.y * sv[q].w);
        }
      }
      __syncwarp();
      if (PARO_DBG(a)) {
        const unsigned long long c = clock64();
        q_par += c - q0;
        q0 = c;
      }
      if (threadIdx.x == 0 && gams[0] == g0) PARO_TL(a, 8);
#pragma unroll
      for (int t = 0; t < 8; ++t) {  // a5: rotations t = 1..L, Eq. 4 form, pre-update values
        if (t >= L_eff) break;
#pragma unroll
        for (int q = 0; q < NG; ++q) {
          const uint32_t i0 = ixr[q][t] & 0xff, j0 = (ixr[q][t] >> 8) & 0xff;
          const uint32_t i1 = (ixr[q][t] >> 16) & 0xff, j1 = ixr[q][t] >> 24;
          const float4 c = csr[q][t];
#pragma unroll
          for (int b = 0; b < BT; ++b) {
            float* sb = scr + (q * BT + b) * 132;
            const float a0 = sb[i0], b0 = sb[j0];
            const float a1 = sb[i1], b1 = sb[j1];
            sb[i0] = c.x * a0 - c.y * b0;
            sb[j0] = c.y * a0 + c.x * b0;
            sb[i1] = c.z * a1 - c.w * b1;
            sb[j1] = c.w * a1 + c.z * b1;
          }
        }
        __syncwarp();
      }
      if (PARO_DBG(a)) {
        const unsigned long long c = clock64();
        q_rot += c - q0;
        q0 = c;
      }
      if (threadIdx.x == 0 && gams[0] == g0) PARO_TL(a, 6);
      if (CL > 1 && !cwaited) {
        cluster_wait();  // every CTA of the cluster is running and initialised: DSMEM is legal
        cwaited = true;
      }
      if constexpr (IM) {
        // IMMA path: x' of (group, token) -> fixed point x'fix = rint(x' * 2^(14 - E)), 2^E >= max|x'|
        // over the group (|x'fix| <= 2^14), split into two balanced s8 digits x'fix = 256 hi + lo.
        // The digits are laid out as IMMA B fragments: slot (group, token, hd = 2 hl + dg, t) holds
        // 16 bytes, byte i of word j = digit dg (0: hi, 1: lo) of the channel in nibble hl of byte i
        // of word j of quad t (tile_layout.cuh).  Per (group, token) also X = sum x'fix (zero-point
        // term) and F = 2^(E - 14).
#pragma unroll
        for (int q = 0; q < NG; ++q) {
          const int gam = gams[q];
          int fxv[BT][4];
          int Xs[BT];
          float Fs[BT];
#pragma unroll
          for (int b = 0; b < BT; ++b) {
            const float4 v = *reinterpret_cast<const float4*>(scr + (q * BT + b) * 132 + 4 * lane);
            float m = fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w)));
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            const uint32_t mb = __float_as_uint(m);
            int E = mb < 0x00800000u ? -100 : static_cast<int>(mb >> 23) - 127 + ((mb & 0x7fffffu) != 0u ? 1 : 0);
            E = max(E, -100);
            const float mul = __uint_as_float(static_cast<uint32_t>(141 - E) << 23);  // 2^(14 - E)
            Fs[b] = __uint_as_float(static_cast<uint32_t>(113 + E) << 23);           // 2^(E - 14)
            fxv[b][0] = __float2int_rn(v.x * mul);
            fxv[b][1] = __float2int_rn(v.y * mul);
            fxv[b][2] = __float2int_rn(v.z * mul);
            fxv[b][3] = __float2int_rn(v.w * mul);
            int xs = (fxv[b][0] + fxv[b][1]) + (fxv[b][2] + fxv[b][3]);
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) xs += __shfl_xor_sync(0xffffffffu, xs, o);
            Xs[b] = xs;
          }
          __syncwarp();  // every lane has read its x' (the digit image overwrites the scratch)
#pragma unroll
          for (int b = 0; b < BT; ++b) {
            uint8_t* img = reinterpret_cast<uint8_t*>(scr + (q * BT + b) * 132);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int c = 4 * lane + e;
              const int j = c >> 5, hl = (c >> 4) & 1, i = ((c & 1) << 1) | ((c >> 3) & 1), tq = (c >> 1) & 3;
              const int fx = fxv[b][e];
              const int lo = static_cast<int>(static_cast<int8_t>(fx & 0xff));
              const int hi = (fx - lo) >> 8;
              img[((hl * 2 + 0) * 4 + tq) * 16 + j * 4 + i] = static_cast<uint8_t>(hi);
              img[((hl * 2 + 1) * 4 + tq) * 16 + j * 4 + i] = static_cast<uint8_t>(lo);
            }
          }
          __syncwarp();
          const int sl = lane & 15, tl = lane >> 4;
          if (tl < BT) {
            const uint4 v =
                *reinterpret_cast<const uint4*>(reinterpret_cast<const uint8_t*>(scr + (q * BT + tl) * 132) + sl * 16);
            const uint32_t uo = u_addr + static_cast<uint32_t>(((gam * BT + tl) * 16 + sl) * 16);
            const uint32_t so = s_addr + static_cast<uint32_t>((gam * 8 + 2 * tl) * 4);
            const int Xt = (BT == 2 && tl) ? Xs[BT - 1] : Xs[0];
            const float Ft = (BT == 2 && tl) ? Fs[BT - 1] : Fs[0];
            if (CL > 1) {
#pragma unroll 1
              for (int r = 0; r < CL; ++r) {
                const uint32_t rb = mapa(bar_addr, r);
                st_async_v4(mapa(uo, r), v, rb);
                if (sl == 0) st_async_v2(mapa(so, r), static_cast<uint32_t>(Xt), __float_as_uint(Ft), rb);
              }
            } else {
              *reinterpret_cast<uint4*>(ufr + (uo - u_addr)) = v;
              if (sl == 0) {
                reinterpret_cast<int*>(xsum)[gam * 8 + 2 * tl] = Xt;
                xsum[gam * 8 + 2 * tl + 1] = Ft;
              }
            }
          }
        }
      } else {
#pragma unroll
      for (int q = 0; q < NG; ++q) {
        const int gam = gams[q];
#pragma unroll
        for (int b = 0; b < BT; ++b) {
          const float2 v01 = lds_f2_a(scr_a + static_cast<uint32_t>((q * BT + b) * 132 + k0) * 4);
          const float2 v89 = lds_f2_a(scr_a + static_cast<uint32_t>((q * BT + b) * 132 + k0 + 8) * 4);
          const uint32_t p0 = pack_half2(v01.x, v01.y);
          const uint32_t p1 = pack_half2(v89.x, v89.y);
          // sum over the group of the fp16-rounded x' (the zero-point term uses exactly the
          // values the tensor cores multiply)
          float cs = half2_sum(p0) + half2_sum(p1);
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) cs += __shfl_xor_sync(0xffffffffu, cs, o);
          const uint32_t uo = u_addr + static_cast<uint32_t>(((gam * 4 + i4) * BT + b) * 64 + t4 * 16 + hf * 8);
          const uint32_t so = s_addr + static_cast<uint32_t>((gam * 8 + b) * 4);
          if (CL > 1) {
#pragma unroll 1
            for (int r = 0; r < CL; ++r) {  // not unrolled: small code (instruction cache)
              const uint32_t rb = mapa(bar_addr, r);
              st_async_v2(mapa(uo, r), p0, p1, rb);
              if (lane == 0) st_async_b32(mapa(so, r), __float_as_uint(cs), rb);
            }
          } else {
            *reinterpret_cast<uint2*>(ufr + (uo - u_addr)) = make_uint2(p0, p1);
            if (lane == 0) xsum[gam * 8 + b] = cs;
          }
        }
      }
      }  // !IM
      __syncwarp();
      if (PARO_DBG(a)) {
        const unsigned long long c = clock64();
        q_out += c - q0;
        q0 = c;
      }
      if (threadIdx.x == 0 && gams[0] == g0) PARO_TL(a, 7);
    };

    // This warp's first two groups: both parameter sets are loaded into registers before the
    // activations arrive (their L2 latency overlaps the activation copy), then both groups are
    // transformed in lockstep.
    const int gams[2] = {g0 + warp, g0 + warp + NW};
    const int ng = gams[1] < g1 ? 2 : (gams[0] < g1 ? 1 : 0);
    float4 cs2[2][8];
    uint32_t ix2[2][8];
    float4 sv2[2];
#pragma unroll
    for (int q = 0; q < 2; ++q)
      if (q < ng) load_params(gams[q], cs2[q], ix2[q], sv2[q]);
    if (ng > 0 && a.pdl) pdl_wait();  // x may be written by the previous kernel on the stream
    // activations of the (up to two) groups -> registers, then let the producer stream weights
    uint2 xr2[2][BT];
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int b = 0; b < BT; ++b)
        xr2[q][b] = (q < ng && b < B) ? __ldg(reinterpret_cast<const uint2*>(static_cast<const uint8_t*>(a.x) +
                                                                             (static_cast<int64_t>(b) * K + gams[q] * GRP + 4 * lane) * 2))
                                      : make_uint2(0u, 0u);  // tokens >= B: x = 0 (x' = 0, never stored)
    if (a.xfirst) named_bar_arrive(2, (NW + 1) * 32);
    if (threadIdx.x == 0) PARO_TL(a, 1);
    // rounds of (up to) two groups; the parameters / activations of later rounds (large K,
    // few CTAs per cluster) are loaded at the top of their round.  One call site per group
    // count keeps a single copy of each transform instance (instruction-cache footprint).
    for (int r = 0;; ++r) {
      int gr[2] = {gams[0] + 2 * r * NW, gams[1] + 2 * r * NW};
      const int nr = gr[1] < g1 ? 2 : (gr[0] < g1 ? 1 : 0);
      if (nr == 0) break;
      if (r > 0) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          if (q < nr) load_params(gr[q], cs2[q], ix2[q], sv2[q]);
#pragma unroll
          for (int b = 0; b < BT; ++b)
            xr2[q][b] = (q < nr && b < B)
                            ? __ldg(reinterpret_cast<const uint2*>(static_cast<const uint8_t*>(a.x) +
                                                                   (static_cast<int64_t>(b) * K + gr[q] * GRP + 4 * lane) * 2))
                            : make_uint2(0u, 0u);
        }
      }
      if (nr == 2)
        process(std::integral_constant<int, 2>{}, gr, cs2, ix2, sv2, xr2);
      else
        process(std::integral_constant<int, 1>{}, gr, cs2, ix2, sv2, xr2);
    }
    if (PARO_DBG(a)) q0 = clock64();
    if (CL > 1) {
      if (!cwaited) cluster_wait();
      mbar_wait(xpbar, 0);  // every group's x' has arrived from its owner CTA
    } else {
      named_bar_sync(1, NW * 32);
    }
    if (PARO_DBG(a) && lane == 0 && blockIdx.x < 1024 && warp < 16) {
      unsigned long long* pp = g_paro_prof + (blockIdx.x * 16 + warp) * 8;
      pp[4] = q_par;
      pp[5] = q_rot;
      pp[6] = q_out;
      pp[7] = clock64() - q0;  // waiting for the cluster's x'
    }
  }
  if (threadIdx.x == 0) PARO_TL(a, 2);

  // ------------------------------------------------------------ phase 2: GEMV on mma.sync
  constexpr int TR = TILE_ROWS;  // 32 rows per tile: two 16-row MMA blocks (rows g, g+8 | g+16, g+24)
  float* pw = part + static_cast<size_t>(warp) * a.R_max * TR * BT;
  for (int i = lane; i < n_rho * TR * BT; i += 32) pw[i] = 0.f;
  __syncwarp();
  const int gq = lane >> 2, t = lane & 3;
  // B-fragment token of this lane: columns >= BT duplicate token BT-1 (computed, never stored)
  const int bq = min(gq, BT - 1);
  const uint32_t u_a = smem_u32(ufr), xs_a = smem_u32(xsum), ring_a = smem_u32(ring);
  // acc[4h + e]: rows gq + 16h (e = 0, 1) and gq + 16h + 8 (e = 2, 3), columns 2t, 2t + 1
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
  int cur = -1;
  // IMMA path: lane (gq, t) accumulates rows gq + 8q (acc[q], q = 0..3) of token tok_l; lanes
  // t = 2 tok_l (low-nibble channels) and t = 2 tok_l + 1 (high-nibble channels) are summed at flush
  const int tok_l = (IM && BT == 2) ? (t >> 1) : 0;
  const int tokB = (IM && BT == 2) ? (gq >> 2) : 0;      // token of the B column this lane supplies
  const uint32_t mlo = ((gq >> 1) & 1) ? 0u : 0xffffffffu;  // column gq carries low-nibble digits
  const uint32_t mhi = ~mlo;
  const int xmask = (t & 1) ? 0 : -1;   // zero-point term on the low-nibble lane only
  const float fsc = (t & 1) ? 0.0625f : 1.0f;  // high-nibble products carry 16 q
  auto flush = [&]() {
    float* pr = pw + cur * TR * BT;
    if constexpr (IM) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float v = acc[q] + __shfl_xor_sync(0xffffffffu, acc[q], 1);
        if ((t & 1) == 0 && (t >> 1) < BT && tok_l < B) pr[(gq + 8 * q) * BT + tok_l] = v;
      }
    } else {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (2 * t < B) {
          pr[(gq + 16 * h) * BT + 2 * t] = acc[4 * h + 0];
          pr[(gq + 16 * h + 8) * BT + 2 * t] = acc[4 * h + 2];
        }
        if (2 * t + 1 < B) {
          pr[(gq + 16 * h) * BT + 2 * t + 1] = acc[4 * h + 1];
          pr[(gq + 16 * h + 8) * BT + 2 * t + 1] = acc[4 * h + 3];
        }
      }
    }
  };
  // this warp's tiles of stage st are tA + st * TPS + warp + NW * m: (row block, group) from
  // one division per stage, then advanced incrementally
  int rb = 0, g = 0;
  unsigned long long c_wait = 0, c_work = 0, c_t = PARO_DBG(a) ? clock64() : 0;
  for (int st = 0; st < n_stages; ++st) {
    const int slot = st % a.S;
    if (st == 0 && threadIdx.x == 0) PARO_TL(a, 10);  // debug: reached the first stage wait
    mbar_wait(&full[slot], (st / a.S) & 1);
    if (PARO_DBG(a)) {
      const unsigned long long c = clock64();
      c_wait += c - c_t;
      c_t = c;
    }
    if (st == 0 && threadIdx.x == 0) PARO_TL(a, 3);
    if (st == n_stages - 1 && threadIdx.x == 0) PARO_TL(a, 11);
    const uint32_t sbase = ring_a + static_cast<uint32_t>(slot) * a.slot_bytes;
    const int nts = min(TPS, n_my - st * TPS);
    {
      const int tl0 = tA + st * TPS + warp;
      rb = tl0 / G;
      g = tl0 - rb * G;
    }
    for (int i = warp; i < nts; i += NW) {
      if (rb - rho_first != cur) {
        if (cur >= 0) flush();
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = 0.f;
        cur = rb - rho_first;
      }
      // codes: quad t of rows gq, gq + 8, gq + 16, gq + 24 (words j = 0..3 each)
      const uint32_t ca = sbase + static_cast<uint32_t>(i) * TILE_CODE_BYTES + lane * 16;
      uint4 w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) w[q] = lds128_a(ca + q * 512);
      if constexpr (IM) {
        // A = codes as u8 (low nibbles: w & 0x0F0F0F0F; high: w & 0xF0F0F0F0 = 16 q), B = x'fix digits.
        // k-steps: (words 0, 1) and (words 2, 3) of the low nibbles into columns of low-nibble digits,
        // then the same words' high nibbles into the high-nibble columns (the other columns see B = 0).
        const uint4 r = lds128_a(u_a + static_cast<uint32_t>((((g * BT + tokB) * 16) + (gq & 3) * 4 + t) * 16));
        constexpr uint32_t ML = 0x0f0f0f0fu, MH = 0xf0f0f0f0u;
        int D[2][4];
#pragma unroll
        for (int h = 0; h < 2; ++h)
          imma_16832_z(D[h], w[2 * h].x & ML, w[2 * h + 1].x & ML, w[2 * h].y & ML, w[2 * h + 1].y & ML, r.x & mlo,
                       r.y & mlo);
#pragma unroll
        for (int h = 0; h < 2; ++h)
          imma_16832(D[h], w[2 * h].z & ML, w[2 * h + 1].z & ML, w[2 * h].w & ML, w[2 * h + 1].w & ML, r.z & mlo,
                     r.w & mlo);
#pragma unroll
        for (int h = 0; h < 2; ++h)
          imma_16832(D[h], w[2 * h].x & MH, w[2 * h + 1].x & MH, w[2 * h].y & MH, w[2 * h + 1].y & MH, r.x & mhi,
                     r.y & mhi);
#pragma unroll
        for (int h = 0; h < 2; ++h)
          imma_16832(D[h], w[2 * h].z & MH, w[2 * h + 1].z & MH, w[2 * h].w & MH, w[2 * h + 1].w & MH, r.z & mhi,
                     r.w & mhi);
        // epilogue (a6): I = sum (q - z) x'fix exactly in int32 (low lane: 256 D_hi + D_lo - z X;
        // high lane: 16x that sum of its channels), y += S * F * I
        const uint2 sp = lds_u64_a(sbase + a.sc_off + static_cast<uint32_t>(i) * TILE_SCALE_BYTES + gq * 8);
        const uint32_t zw = lds_u16z_a(sbase + a.z_off + static_cast<uint32_t>(i) * TILE_ZERO_BYTES + gq * 2);
        const uint2 mt = lds_u64_a(xs_a + static_cast<uint32_t>((g * 8 + 2 * tok_l) * 4));
        const int Xl = static_cast<int>(mt.x) & xmask;
        const float Fl = __uint_as_float(mt.y) * fsc;
        const float2 Sa = __half22float2(*reinterpret_cast<const __half2*>(&sp.x));  // rows gq, gq + 8
        const float2 Sb = __half22float2(*reinterpret_cast<const __half2*>(&sp.y));  // rows gq + 16, gq + 24
        const float Sr[4] = {Sa.x, Sa.y, Sb.x, Sb.y};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int zq = static_cast<int>((zw >> (4 * q)) & 15u);
          const int h = q >> 1, e = (q & 1) * 2;
          const int I = D[h][e] * 256 + D[h][e + 1] - zq * Xl;
          acc[q] = fmaf(static_cast<float>(I), Sr[q] * Fl, acc[q]);
        }
      } else {
      // B fragments of group g (token bq): registers 4 * ii .. 4 * ii + 3 = MMAs 2 ii, 2 ii + 1
      uint32_t bf[16];
      {
        const uint32_t xa = u_a + static_cast<uint32_t>(((g * 4) * BT + bq) * 64 + t * 16);
#pragma unroll
        for (int ii = 0; ii < 4; ++ii) {
          const uint4 v = lds128_a(xa + ii * BT * 64);
          bf[4 * ii + 0] = v.x;
          bf[4 * ii + 1] = v.y;
          bf[4 * ii + 2] = v.z;
          bf[4 * ii + 3] = v.w;
        }
      }
      // 2^-24 sum q x' (low-nibble MMAs) and 2^-20 sum q x' (high-nibble MMAs) per 16-row block
      float D1[2][4], D16[2][4];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t w0[4] = {w[2 * h].x, w[2 * h].y, w[2 * h].z, w[2 * h].w};
        const uint32_t w1[4] = {w[2 * h + 1].x, w[2 * h + 1].y, w[2 * h + 1].z, w[2 * h + 1].w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t x = w0[j], y = w1[j], x8 = x >> 8, y8 = y >> 8;
          if (j == 0) {
            mma_16816_z(D1[h], x & 0x000F000Fu, y & 0x000F000Fu, x8 & 0x000F000Fu, y8 & 0x000F000Fu, bf[0], bf[1]);
            mma_16816_z(D16[h], x & 0x00F000F0u, y & 0x00F000F0u, x8 & 0x00F000F0u, y8 & 0x00F000F0u, bf[2],
                        bf[3]);
          } else {
            mma_16816(D1[h], x & 0x000F000Fu, y & 0x000F000Fu, x8 & 0x000F000Fu, y8 & 0x000F000Fu, bf[4 * j],
                      bf[4 * j + 1]);
            mma_16816(D16[h], x & 0x00F000F0u, y & 0x00F000F0u, x8 & 0x00F000F0u, y8 & 0x00F000F0u, bf[4 * j + 2],
                      bf[4 * j + 3]);
          }
        }
      }
      // epilogue of the tile (a6): y += S * (2^24 * (D1 + D16 / 16) - z * sum x')
      const uint2 sp = lds_u64_a(sbase + a.sc_off + static_cast<uint32_t>(i) * TILE_SCALE_BYTES + gq * 8);
      const uint32_t zw = lds_u16z_a(sbase + a.z_off + static_cast<uint32_t>(i) * TILE_ZERO_BYTES + gq * 2);
      const float2 Sa = __half22float2(*reinterpret_cast<const __half2*>(&sp.x));  // rows gq, gq + 8
      const float2 Sb = __half22float2(*reinterpret_cast<const __half2*>(&sp.y));  // rows gq + 16, gq + 24
      const float2 X2 = lds_f2_a(xs_a + static_cast<uint32_t>((g * 8 + 2 * t) * 4));
      const float Sr[4] = {Sa.x, Sa.y, Sb.x, Sb.y};
#pragma unroll
      for (int q = 0; q < 4; ++q) {  // row gq + 8q: block h = q / 2, fragment half q % 2
        const float zq = static_cast<float>((zw >> (4 * q)) & 15u);
        const int h = q >> 1, e = (q & 1) * 2;
        acc[4 * h + e] = fmaf(Sr[q], fmaf(fmaf(D16[h][e], 0.0625f, D1[h][e]), TWO_P24, -zq * X2.x), acc[4 * h + e]);
        if (BT > 1)  // column 2t + 1 holds a token only when BT > 1
          acc[4 * h + e + 1] =
              fmaf(Sr[q], fmaf(fmaf(D16[h][e + 1], 0.0625f, D1[h][e + 1]), TWO_P24, -zq * X2.y), acc[4 * h + e + 1]);
      }
      }  // !IM
      g += NW;
      while (g >= G) {
        g -= G;
        ++rb;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);  // this warp is done with the stage
    if (PARO_DBG(a)) {
      const unsigned long long c = clock64();
      c_work += c - c_t;
      c_t = c;
    }
  }
  if (PARO_DBG(a) && lane == 0 && blockIdx.x < 1024 && warp < 16) {
    unsigned long long* pp = g_paro_prof + (blockIdx.x * 16 + warp) * 8;
    pp[0] = c_wait;
    pp[1] = c_work;
    pp[2] = static_cast<unsigned long long>(n_stages);
    pp[3] = static_cast<unsigned long long>(n_my);
  }
  if (cur >= 0) flush();
  if (threadIdx.x == 0) PARO_TL(a, 4);
  if (a.pdl) pdl_wait();  // y may still be read by the previous kernel (no-op once it has finished)

  // ------------------------------------------------------------ reduction + epilogue (a8)
  named_bar_sync(1, NW * 32);
  const int n_out = n_rho * TR * BT;
  for (int idx = threadIdx.x; idx < n_out; idx += NW * 32) {
    const int rho = idx / (TR * BT), r = (idx / BT) % TR, b = idx % BT;
    if (b >= B) continue;
    // fixed-order sum over the warps (four independent chains, then combined: deterministic)
    const float* pp = part + (static_cast<size_t>(rho) * TR + r) * BT + b;
    const size_t wstride = static_cast<size_t>(a.R_max) * TR * BT;
    float s4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
    for (int w = 0; w < NW; ++w) s4[w & 3] += pp[w * wstride];
    float sum = (s4[0] + s4[1]) + (s4[2] + s4[3]);
    const int rg = rho_first + rho;
    if (rho == 0 && !own_first) {
      // the block started in an earlier CTA: push this partial to it (recv slot crank - owner - 1)
      const int owner = cta_of_tile(rg * G, nt, lcl);
      const uint32_t dst =
          smem_u32(recv) + static_cast<uint32_t>((((crank - owner - 1) * TR + r) * BT + b) * 4);
      st_async_b32(mapa(dst, owner), __float_as_uint(sum), mapa(smem_u32(rbar), owner));
    } else if (rho == n_rho - 1 && last_cta > crank) {
      part[(static_cast<size_t>(rho) * TR + r) * BT + b] = sum;  // warp-0 slot of this element
    } else {
      const int64_t n = static_cast<int64_t>(rbc0 + rg) * TR + r;
      if (n < d.N) {
        float v = sum;
        if (d.bias) v += __ldg(d.bias + n);
        store_out(d.y, a.y_dtype, static_cast<int64_t>(b) * d.N + n, v);
      }
    }
  }
  if (last_cta > crank) {
    named_bar_sync(1, NW * 32);
    mbar_wait(rbar, 0);
    const int rho = n_rho - 1, rg = rho_first + rho;
    for (int idx = threadIdx.x; idx < TR * BT; idx += NW * 32) {
      const int r = idx / BT, b = idx % BT;
      if (b >= B) continue;
      float sum = part[(static_cast<size_t>(rho) * TR + r) * BT + b];
      for (int c = crank + 1; c <= last_cta; ++c)  // fixed order
        if (cta_tile_start(c + 1, nt, lcl) > cta_tile_start(c, nt, lcl)) sum += recv[((c - crank - 1) * TR + r) * BT + b];
      const int64_t n = static_cast<int64_t>(rbc0 + rg) * TR + r;
      if (n < d.N) {
        float v = sum;
        if (d.bias) v += __ldg(d.bias + n);
        store_out(d.y, a.y_dtype, static_cast<int64_t>(b) * d.N + n, v);
      }
    }
  }
  if (threadIdx.x == 0) PARO_TL(a, 5);
}

#if PARO_ENABLE_DEBUG
extern "C" int paro_debug_read_prof(unsigned long long* host, int n) {
  if (n > 1024 * 16 * 8) n = 1024 * 16 * 8;
  return static_cast<int>(cudaMemcpyFromSymbol(host, g_paro_prof, sizeof(unsigned long long) * n));
}

// debug: copy the per-CTA event timeline (ns, %globaltimer) of the last debug launch
extern "C" int paro_debug_read_timeline(unsigned long long* host, int n) {
  if (n > 1024 * TL_EVENTS) n = 1024 * TL_EVENTS;
  return static_cast<int>(cudaMemcpyFromSymbol(host, g_paro_timeline, sizeof(unsigned long long) * n));
}
#endif

// ============================================================================ host side
static int smem_optin() { return device_smem_optin(); }

static inline uint32_t align_up(uint32_t v, uint32_t a) { return (v + a - 1) / a * a; }

static const void* kernel_for(int BT, int threads, bool im) {
#define PARO_KF(BT_, IM_)                                                                          \
  if (BT == BT_ && im == IM_) {                                                                   \
    if (threads <= 288) return reinterpret_cast<const void*>(&paro_gemv_kernel<BT_, 288, IM_>); \
    if (threads <= 512) return reinterpret_cast<const void*>(&paro_gemv_kernel<BT_, 512, IM_>); \
    if (threads <= 640) return reinterpret_cast<const void*>(&paro_gemv_kernel<BT_, 640, IM_>); \
  }
  PARO_KF(1, false)
  PARO_KF(2, false)
  PARO_KF(4, false)
  PARO_KF(8, false)
  PARO_KF(1, true)
  PARO_KF(2, true)
#undef PARO_KF
  return nullptr;
}

// Co-resident CTAs for this launch shape (whole clusters), from the occupancy API.
static int max_resident_ctas(int BT, int threads, int smem, int CL, bool im) {
  const void* k = kernel_for(BT, threads, im);
  if (!k) return 0;
  if (ensure_smem_attr(k, smem) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  if (CL > 1) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(CL * 64);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = CL;
    at.val.clusterDim.y = 1;
    at.val.clusterDim.z = 1;
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, k, &cfg) != cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
    return nc * CL;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, threads, smem) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return per_sm * device_sm_count();
}

// Plan overrides for experiments exist only in builds with -DPARO_DEBUG_KNOBS=1 (never in
// the shipped library: a stray environment variable must not change what a call computes).
static int env_int(const char* name, int dflt) {
#if PARO_DEBUG_KNOBS
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
#else
  (void)name;
  return dflt;
#endif
}

static bool plan_try(int B, int n_lin, const int64_t* Ns, const int* Ls, int64_t K, int rotate, int NW, int ctas_pref,
                     int CL, int TPS_req, int min_stages, GemvConfig* cfg, const char** why) {
  GemvConfig c{};
  if (n_lin < 1 || n_lin > GEMV_MAX_LIN) {
    *why = "1..4 linears per decode launch";
    return false;
  }
  if (B != 1 && B != 2 && B != 4 && B != 8) {
    *why = "decode token tile must be 1, 2, 4 or 8";
    return false;
  }
  c.BT = B;
  // integer tensor-core path (x' as 16-bit fixed point per group) for 1-2 tokens; PARO_IMMA=0: fp16 HMMA
  c.IM = B <= 2 && env_int("PARO_IMMA", 1) != 0;
  int64_t NBsum = 0;
  int L = 0;
  int64_t NB[GEMV_MAX_LIN];
  for (int i = 0; i < n_lin; ++i) {
    NB[i] = (Ns[i] + TILE_ROWS - 1) / TILE_ROWS;
    NBsum += NB[i];
    L = std::max(L, Ls[i]);
  }
  const int G = static_cast<int>(K / GRP);
  int ctas_per_sm = (NW <= 8 && ctas_pref == 2) ? 2 : 1;
  // co-resident mode: one CTA per SM in the grid, but a half-SM footprint (smem, registers) so
  // that the next launch on the stream (PDL) is resident while this one runs
  const bool coloc = ctas_pref == 3 && NW <= 8;
  if (coloc) ctas_per_sm = 2;
  while (CL > 1 && CL > G) CL /= 2;
  const int TPS = std::max(1, std::min(64, TPS_req > 0 ? TPS_req : 2 * NW));
  c.NW = NW;
  c.CL = CL;
  c.a.xfirst = env_int("PARO_XFIRST", 1);           // weights wait until the transform loads are out
  c.a.early_stages = env_int("PARO_EARLY_STAGES", 2);  // under PDL: stages requested before that
  c.a.stagger = env_int("PARO_STAGGER", 1);  // first stage lands before the rest of the ring is requested
  GemvArgs& a = c.a;
  a.n_lin = n_lin;
  a.B = B;
  a.K = static_cast<int>(K);
  a.G = G;
  a.rotate = rotate;
  a.NW = NW;
  a.TPS = TPS;
  a.sc_off = static_cast<uint32_t>(TPS) * TILE_CODE_BYTES;
  a.z_off = a.sc_off + static_cast<uint32_t>(TPS) * TILE_SCALE_BYTES;
  a.slot_bytes = align_up(a.z_off + static_cast<uint32_t>(TPS) * TILE_ZERO_BYTES, 128);
  const int threads = (NW + 1) * 32;
  const uint32_t u_bytes = align_up(static_cast<uint32_t>(B) * K * 2, 128);
  const uint32_t xs_bytes = align_up(static_cast<uint32_t>(G) * 8 * 4, 128);
  const int g_per = (G + CL - 1) / CL;
  // transform scratch of the warps that own groups (two groups in lockstep when g_per > NW)
  a.scr_groups = g_per > NW ? 2 : 1;
  const uint32_t scr_bytes =
      align_up(static_cast<uint32_t>(std::min(NW, g_per)) * a.scr_groups * B * 132 * 4, 128);
  const uint32_t recv_bytes = align_up(static_cast<uint32_t>(std::max(1, CL - 1)) * TILE_ROWS * B * 4, 128);
  if (u_bytes > 64 * 1024) ctas_per_sm = 1;
  int budget = (smem_optin() + 1024) / ctas_per_sm - 2048;
  int max_tiles_cta = 0;
  // split the grid's clusters over the linears in proportion to their row blocks (>= 1 each,
  // never more clusters than row blocks)
  auto split = [&](int grid) -> bool {
    int ncl = grid / CL;
    if (ncl < n_lin) return false;
    if (ncl > NBsum) ncl = static_cast<int>(NBsum);
    int cl[GEMV_MAX_LIN], used = 0, big = 0;
    for (int i = 0; i < n_lin; ++i) {
      cl[i] = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(NB[i], ncl * NB[i] / NBsum)));
      used += cl[i];
      if (NB[i] > NB[big]) big = i;
    }
    cl[big] = static_cast<int>(std::min<int64_t>(NB[big], cl[big] + std::max(0, ncl - used)));
    int begin = 0;
    max_tiles_cta = 0;
    for (int i = 0; i < n_lin; ++i) {
      GemvLinear& d = a.lin[i];
      d.N = static_cast<int>(Ns[i]);
      d.L = Ls[i];
      d.cta_begin = begin;
      d.n_ctas = cl[i] * CL;
      d.rb_base = static_cast<int>(NB[i] / cl[i]);
      d.rb_extra = static_cast<int>(NB[i] % cl[i]);
      const int nt_max = (d.rb_base + (d.rb_extra ? 1 : 0)) * G;
      max_tiles_cta = std::max(max_tiles_cta, (nt_max + CL - 1) / CL);
      begin += d.n_ctas;
    }
    c.grid = begin;
    return true;
  };
  auto layout = [&](int grid) -> bool {
    if (!split(grid)) return false;
    a.R_max = (max_tiles_cta + G - 1) / G + 1;
    uint32_t off = 0;
    a.off_u = off;
    off += u_bytes;
    a.off_xs = off;
    off += xs_bytes;
    a.off_scr = off;
    off += scr_bytes;
    a.off_part = off;
    off += align_up(static_cast<uint32_t>(NW) * a.R_max * TILE_ROWS * B * 4, 128);
    a.off_recv = off;
    off += recv_bytes;
    a.off_bar = off;
    off += 64 * 16;  // up to 60 stages x (full, empty) + 3 singles
    a.off_ring = align_up(off, 1024);
    const int64_t ring_avail = static_cast<int64_t>(budget) - a.off_ring;
    int S = static_cast<int>(ring_avail / a.slot_bytes);
    const int stages_needed = std::max(1, (max_tiles_cta + TPS - 1) / TPS);
    if (S > stages_needed) S = stages_needed;
    if (S > 60) S = 60;
    if (S < std::max(1, std::min(min_stages, stages_needed))) return false;
    a.S = S;
    a.smem_total = a.off_ring + static_cast<uint32_t>(S) * a.slot_bytes;
    return true;
  };
  int grid = device_sm_count() * (coloc ? 1 : ctas_per_sm) / CL * CL;
  if (grid < CL * n_lin) grid = CL * n_lin;
  if (!layout(grid) && ctas_per_sm == 2) {  // too big for two CTAs per SM: one, with the full budget
    ctas_per_sm = 1;
    budget = smem_optin() - 1024;
    grid = std::max(CL * n_lin, device_sm_count() / CL * CL);
  }
  for (int iter = 0; iter < 3; ++iter) {
    if (grid < CL * n_lin) grid = CL * n_lin;
    if (!layout(grid)) {
      *why = "decode kernel shared-memory plan does not fit";
      return false;
    }
    int resident = max_resident_ctas(c.BT, threads, static_cast<int>(a.smem_total), CL, c.IM);
    if (coloc) resident /= 2;
    if (resident <= 0 || resident >= c.grid) break;
    grid = resident / CL * CL;  // never launch more than one wave
  }
  if (!layout(grid)) {
    *why = "decode kernel shared-memory plan does not fit";
    return false;
  }
  if (env_int("PARO_PLAN_DEBUG", 0))
    fprintf(stderr, "[paro gemv plan] B=%d n_lin=%d K=%lld grid=%d CL=%d NW=%d TPS=%d S=%d R_max=%d smem=%u\n", B,
            n_lin, static_cast<long long>(K), c.grid, CL, NW, TPS, a.S, a.R_max, a.smem_total);
  *cfg = c;
  return true;
}

bool plan_gemv(int B, int n_lin, const int64_t* Ns, const int* Ls, int64_t K, int rotate, GemvConfig* cfg,
               const char** why) {
  // Default: 15 compute warps, 1 CTA / SM, clusters of 4, 2 tiles per warp per stage (measured
  // best on the bench's Llama-3-8B layer); PARO_NW / PARO_CTAS_PER_SM / PARO_CLUSTER / PARO_TPS
  // override.  Shapes whose shared-memory plan does not fit fall back to 8 warps.
  const int NW = std::max(1, std::min(19, env_int("PARO_NW", 15)));
  const int cps_env = env_int("PARO_CTAS_PER_SM", 2);
  const int cps = cps_env == 1 ? 1 : (cps_env == 3 ? 3 : 2);
  // clusters of 4 share the transform 4 ways; very large launches with few groups (gate/up at
  // K = 4096) prefer pairs, which tile all 148 SMs (clusters of 4 leave 16 idle)
  int64_t tiles = 0;
  for (int i = 0; i < n_lin; ++i) tiles += (Ns[i] + TILE_ROWS - 1) / TILE_ROWS * (K / GRP);
  int CL = env_int("PARO_CLUSTER", (K / GRP <= 32 && tiles >= 150LL * device_sm_count()) ? 2 : 4);
  if (CL != 1 && CL != 2 && CL != 4 && CL != 8) CL = 4;
  const int TPS = env_int("PARO_TPS", 0);
  // prefer >= 2 ring stages (large token tiles eat shared memory: halve the stage first)
  if (plan_try(B, n_lin, Ns, Ls, K, rotate, NW, cps, CL, TPS, 2, cfg, why)) return true;
  if (plan_try(B, n_lin, Ns, Ls, K, rotate, NW, cps, CL, NW, 2, cfg, why)) return true;
  if (plan_try(B, n_lin, Ns, Ls, K, rotate, NW, cps, CL, NW, 1, cfg, why)) return true;
  if (NW > 8 && plan_try(B, n_lin, Ns, Ls, K, rotate, 8, 2, CL, 0, 1, cfg, why)) return true;
  return plan_try(B, n_lin, Ns, Ls, K, rotate, 4, 1, CL, 0, 1, cfg, why);
}

template <int BT, int T, bool IM>
static cudaError_t launch_t(const GemvConfig& c, cudaStream_t st) {
  auto kern = paro_gemv_kernel<BT, T, IM>;
  cudaError_t e0 = ensure_smem_attr(reinterpret_cast<const void*>(kern), static_cast<int>(c.a.smem_total));
  if (e0 != cudaSuccess) return e0;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(c.grid);
  cfg.blockDim = dim3((c.NW + 1) * 32);
  cfg.dynamicSmemBytes = c.a.smem_total;
  cfg.stream = st;
  cudaLaunchAttribute attrs[2];
  int na = 0;
  if (c.CL > 1) {
    attrs[na].id = cudaLaunchAttributeClusterDimension;
    attrs[na].val.clusterDim.x = c.CL;
    attrs[na].val.clusterDim.y = 1;
    attrs[na].val.clusterDim.z = 1;
    ++na;
  }
  if (c.a.pdl) {
    attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attrs;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, c.a);
}

cudaError_t launch_gemv(const GemvConfig& c, cudaStream_t st) {
  if (c.a.B < 1 || c.a.B > c.BT) return cudaErrorInvalidValue;
  const int threads = (c.NW + 1) * 32;
#define PARO_LG(BT_, IM_)                                          \
  if (c.BT == BT_ && c.IM == IM_) {                                \
    if (threads <= 288) return launch_t<BT_, 288, IM_>(c, st);     \
    if (threads <= 512) return launch_t<BT_, 512, IM_>(c, st);     \
    if (threads <= 640) return launch_t<BT_, 640, IM_>(c, st);     \
  }
  PARO_LG(1, false)
  PARO_LG(2, false)
  PARO_LG(4, false)
  PARO_LG(8, false)
  PARO_LG(1, true)
  PARO_LG(2, true)
#undef PARO_LG
  return cudaErrorInvalidConfiguration;
}

}  // namespace paro
