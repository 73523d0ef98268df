// gemv.cu -- decode path (B <= 4 tokens per launch): scale + L Givens layers fused
// into the activation staging, then the group-wise INT4 dequant GEMV.
//
// SURVEY.md 8(a) rows a4 (stage + scale), a5 (L rotations, Eq. 5 in column form),
// a6 (dequant GEMV), a8 (epilogue).  One kernel, launched as clusters of CL CTAs
// (1-2 CTAs per SM, one wave):
//
//  * producer warp: bulk-copies (cp.async.bulk, TMA engine) first the activations
//    this CTA transforms, then its contiguous row slice of the packed weight (INT4
//    codes / fp16 scales / uint4 zeros, row-major) through a ring of shared-memory
//    stages (SR rows each), completion tracked by mbarriers.
//  * compute warps, phase 1 (transform; PAPER.md:195-209's token / group / pair
//    parallelism): the CL CTAs of a cluster split the K/128 groups; a warp owns a
//    group, keeps its L rotations' (cos, sin, i, j) in registers (loaded before the
//    producer starts, so they do not queue behind the weight stream), stages the
//    group in shared memory, scales by s and applies the L independent rotations
//    (2 pairs per lane per rotation, sync-free inside a rotation, __syncwarp
//    between rotations).  The fp16 x' of the group -- stored with each 8-channel
//    block in (0,4,1,5,2,6,3,7) order, the register order the dequantiser wants --
//    and its 32-channel partial sums go to every CTA of the cluster with st.async
//    (DSMEM), completion counted in bytes on the receiver's mbarrier.  x' never
//    goes to HBM.
//  * compute warps, phase 2 (GEMV): warp wk owns a 512*J-wide K slice; half-warp h
//    handles row 2p+h of each row pair, lane 32*J consecutive K (one 128-group).
//    x' lives in registers as fp16 pairs.  Codes are dequantised in registers with
//    one AND mask per pair of weights: a nibble q in bits [0,4) of an fp16 half IS
//    the subnormal q*2^-24, in bits [4,8) it is 16q*2^-24; fma.rn.f32.f16 (FHFMA)
//    multiplies-accumulates those into fp32, exactly scaled by powers of two.
//    Per (row, group): y += S * (sum q x' - z * sum x').  Row partials are reduced
//    by a transpose-shuffle over the 16 lanes of a half-warp (eight row pairs per
//    stage) and across K-slice warps through shared memory in a fixed order
//    (deterministic).
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "paro_internal.h"
#include "ptx.cuh"

namespace paro {

constexpr int GRP = 128;
constexpr float TWO_M24 = 5.9604644775390625e-08f;  // 2^-24
constexpr float TWO_P24 = 16777216.0f;              // 2^24
constexpr int RP_PER_STAGE = 8;                     // max row pairs per stage (SR <= 16 rows)
constexpr int TL_EVENTS = 12;                        // debug timeline: events per CTA

__device__ unsigned long long g_paro_timeline[1024 * TL_EVENTS];

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define PARO_TL(a, ev)                                                                             \
  do {                                                                                             \
    if ((a).debug && blockIdx.x < 1024) g_paro_timeline[blockIdx.x * TL_EVENTS + (ev)] = gtimer(); \
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

// One 32-bit code word (8 nibbles, k = 8m..8m+7) against the x' pairs
// P[0]=(k0,k4), P[1]=(k1,k5), P[2]=(k2,k6), P[3]=(k3,k7): low nibbles carry q*2^-24
// (chain tl), high nibbles 16q*2^-24 (chain th, scaled by 1/16 at the end, exactly).
__device__ __forceinline__ void dot_word(uint32_t x, const uint32_t* P, float& tl, float& th) {
  const uint32_t x8 = x >> 8;
  tl = fma_f16lo(x & 0x000F000Fu, P[0], tl);
  th = fma_f16lo(x & 0x00F000F0u, P[1], th);
  tl = fma_f16hi(x & 0x000F000Fu, P[0], tl);
  th = fma_f16hi(x & 0x00F000F0u, P[1], th);
  tl = fma_f16lo(x8 & 0x000F000Fu, P[2], tl);
  th = fma_f16lo(x8 & 0x00F000F0u, P[3], th);
  tl = fma_f16hi(x8 & 0x000F000Fu, P[2], tl);
  th = fma_f16hi(x8 & 0x00F000F0u, P[3], th);
}

// MAXT: 288 (<= 8 compute warps) or 544 (<= 16 compute warps, very large K);
// u' occupies 16*J*BT registers per thread (BT * J <= 4).
template <int BT, int J, int MAXT>
__global__ void __launch_bounds__(MAXT, (MAXT <= 288 && BT == 1) ? 2 : 1) paro_gemv_kernel(const GemvArgs a) {
  constexpr int RP = RP_PER_STAGE / J;  // row pairs per stage: SR = 2 * RP rows
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int WK = a.WK;
  const int n_compute_warps = WK * a.RG;
  const bool is_producer = warp == n_compute_warps;
  // which linear this CTA serves (CTA ranges are whole clusters)
  int li = 0;
  while (li + 1 < a.n_lin && static_cast<int>(blockIdx.x) >= a.lin[li + 1].cta_begin) ++li;
  const GemvLinear& d = a.lin[li];
  const int K = a.K, G = a.G, L = d.L;
  const int ZB = (G + 1) >> 1;
  const int SR = a.SR;
  const int NCH = K / 32;  // 32-channel chunks

  __half* u16 = reinterpret_cast<__half*>(smem + a.off_u);          // x' [BT][K], perm8 order
  float* usum = reinterpret_cast<float*>(smem + a.off_usum);         // 2^-24 * chunk sums [BT][NCH]
  uint8_t* xs = smem + a.off_x;                                       // raw x slice [BT][x_cols]
  float* part = reinterpret_cast<float*>(smem + a.off_part);
  uint8_t* ring = smem + a.off_ring;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.off_bar);
  uint64_t* empty = full + a.S;
  uint64_t* xbar = empty + a.S;  // raw activations landed (bulk copy)
  uint64_t* xpbar = xbar + 1;    // x' of all K landed (DSMEM st.async from the cluster)
  uint64_t* pbar = xpbar + 1;    // rotation parameters + s of this CTA's groups landed
  uint64_t* pfree = pbar + 1;    // phase 1 done with them (their ring slots can be refilled)

  const int cta = static_cast<int>(blockIdx.x) - d.cta_begin;
  const int n_rows = d.rows_base + (cta < d.rows_extra ? 1 : 0);
  const int row_begin = cta * d.rows_base + min(cta, d.rows_extra);
  const int n_stages = (n_rows + SR - 1) / SR;
  const uint32_t CL = cluster_nctarank();
  const uint32_t crank = cluster_ctarank();
  // groups whose transform this CTA computes
  const int g_per = (G + static_cast<int>(CL) - 1) / static_cast<int>(CL);
  const int g0 = min(G, static_cast<int>(crank) * g_per);
  const int g1 = min(G, g0 + g_per);
  const int x_cols = (g1 - g0) * GRP;  // activation columns this CTA stages
  const uint32_t x_row_bytes = static_cast<uint32_t>(x_cols) * 2;
  // rotation parameters of groups [g0, g1) (lane-major records, contiguous per group) and
  // s are bulk-copied into the LAST P ring slots before anything else; those slots get
  // weights only after phase 1 has released them (pfree).
  const int L_eff = a.rotate ? L : 0;
  const uint32_t p_cs_bytes = static_cast<uint32_t>(g1 - g0) * 32 * L_eff * 16;
  const uint32_t p_ix_bytes = static_cast<uint32_t>(g1 - g0) * 32 * L_eff * 4;
  const uint32_t p_s_bytes = a.rotate ? static_cast<uint32_t>(x_cols) * 4 : 0;
  // staged parameters: in a dedicated region (param_slots < 0) or in the last
  // param_slots ring slots (lent until phase 1 is done); 0: read from global memory
  const bool pded = a.param_slots < 0;
  const int P = pded ? 0 : a.param_slots;  // lent ring slots
  const bool pstaged = a.param_slots != 0;
  uint8_t* pslot = pded ? smem + a.off_param : ring + static_cast<size_t>(a.S - P) * a.slot_bytes;

  if (threadIdx.x == 0) {
    PARO_TL(a, 0);
    for (int i = 0; i < a.S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], WK);  // a stage is consumed by the WK warps of one row group
    }
    mbar_init(xbar, 1);
    mbar_init(xpbar, 1);
    mbar_init(pbar, 1);
    mbar_init(pfree, n_compute_warps);
    if (CL > 1) mbar_arrive_expect_tx(xpbar, static_cast<uint32_t>(BT) * (K * 2 + NCH * 4));
    fence_mbar_init();
  }
  if (CL > 1) {
    cluster_arrive();
    cluster_wait();  // mbarriers initialised; every CTA of the cluster is running (DSMEM legal)
  } else {
    __syncthreads();
  }
  // Let the next kernel on the stream launch now: its CTAs take SM slots as ours retire
  // and run their prologue (parameter loads) early; its griddepcontrol.wait still
  // orders every access to data this kernel produces.
  if (a.pdl) pdl_launch_dependents();

  // ------------------------------------------------------------ producer warp
  if (is_producer) {
    // Request order (latency-critical first): the compute warps' rotation-parameter
    // loads (handshake on barrier 2), then -- after the PDL wait -- the activations,
    // then the weight ring.  Stages [0, S) need no slot release.
    named_bar_sync(2, (n_compute_warps + 1) * 32);
    const uint64_t pol = l2_evict_first_policy();
    auto issue = [&](int st, int slot) {
      const int r0 = row_begin + st * SR;
      const int nr = min(SR, n_rows - st * SR);
      uint8_t* dst = ring + static_cast<size_t>(slot) * a.slot_bytes;
      const uint32_t cb = static_cast<uint32_t>(nr) * (K / 2);
      const int64_t s_lo = (static_cast<int64_t>(r0) * 2 * G) & ~int64_t(15);
      const int64_t s_hi = (static_cast<int64_t>(r0 + nr) * 2 * G + 15) & ~int64_t(15);
      const int64_t z_lo = (static_cast<int64_t>(r0) * ZB) & ~int64_t(15);
      const int64_t z_hi = (static_cast<int64_t>(r0 + nr) * ZB + 15) & ~int64_t(15);
      const uint32_t sb = static_cast<uint32_t>(s_hi - s_lo), zb = static_cast<uint32_t>(z_hi - z_lo);
      mbar_arrive_expect_tx(&full[slot], cb + sb + zb);
      bulk_g2s(dst, d.codes + static_cast<int64_t>(r0) * (K / 2), cb, &full[slot], pol);
      bulk_g2s(dst + a.sc_off, d.scales + s_lo, sb, &full[slot], pol);
      bulk_g2s(dst + a.z_off, d.zeros + z_lo, zb, &full[slot], pol);
    };
    const int first = min(a.S - P, n_stages);
    if (lane == 0 && pstaged && x_cols > 0 && L_eff > 0) {
      // rotation parameters and s: independent of the previous kernel, latency-critical
      mbar_arrive_expect_tx(pbar, p_cs_bytes + p_ix_bytes + p_s_bytes);
      bulk_g2s_nohint(pslot, reinterpret_cast<const uint8_t*>(d.rot_cs) + static_cast<size_t>(g0) * 32 * L_eff * 16,
                      p_cs_bytes, pbar);
      bulk_g2s_nohint(pslot + p_cs_bytes,
                      reinterpret_cast<const uint8_t*>(d.rot_idx) + static_cast<size_t>(g0) * 32 * L_eff * 4,
                      p_ix_bytes, pbar);
      bulk_g2s_nohint(pslot + p_cs_bytes + p_ix_bytes, d.svec + g0 * GRP, p_s_bytes, pbar);
    }
    if (a.pdl) pdl_wait();  // x may be produced by the previous kernel on the stream
    if (lane == 0) {
      if (x_cols > 0) {
        mbar_arrive_expect_tx(xbar, x_row_bytes * static_cast<uint32_t>(a.B));
        for (int b = 0; b < a.B; ++b)
          bulk_g2s_nohint(xs + static_cast<size_t>(b) * x_row_bytes,
                          static_cast<const uint8_t*>(a.x) + (static_cast<int64_t>(b) * K + g0 * GRP) * 2,
                          x_row_bytes, xbar);
      }
      for (int st = 0; st < first; ++st) issue(st, st);
      // the lent slots: first use once phase 1 released them, then the normal ring
      int st = first;
      if (P > 0) {
        mbar_wait(pfree, 0);
        for (; st < min(a.S, n_stages); ++st) issue(st, st);
      }
      // stages >= S reuse the slot of stage st - S (same row group: S % RG == 0)
      const int RGN = a.RG, SP = a.S / RGN;
      for (; st < n_stages; ++st) {
        const int use = st / RGN;
        const int slot = st % RGN + RGN * (use % SP);
        mbar_wait(&empty[slot], ((use / SP) & 1) ^ 1);  // stage st - S released by its row group
        issue(st, slot);
      }
    }
    __syncwarp();
    return;
  }

  // ------------------------------------------------------------ phase 1: activation transform
  {
    float* scr = reinterpret_cast<float*>(smem + a.off_scr) + warp * (BT * 132);
    const uint32_t u_addr = smem_u32(u16), s_addr = smem_u32(usum), bar_addr = smem_u32(xpbar);
    const int b8 = (lane >> 1) * 8, hh = lane & 1;  // output: lane writes half hh of 8-block b8
    const int c0 = b8 + 2 * hh;
    bool first = true;
    for (int gam = g0 + warp; gam < g1 || first; gam += n_compute_warps) {
      const bool have = gam < g1;
      // rotation parameters of this group -> registers (independent of the previous kernel)
      // records [group][t][32 lanes]: (cos0, sin0, cos1, sin1) and (i0, j0, i1, j1)
      float4 csr[8];
      uint32_t ixr[8];
      float sv[4];
      if (first) {
        named_bar_arrive(2, (n_compute_warps + 1) * 32);  // let the producer start
        if (pstaged && x_cols > 0 && L_eff > 0) mbar_wait(pbar, 0);
        if (x_cols > 0) mbar_wait(xbar, 0);
        if (threadIdx.x == 0) PARO_TL(a, 1);
        first = false;
      }
      if (have && L_eff > 0) {
        if (pstaged) {  // staged in shared memory, records [group][t][32 lanes]
          const float4* csp = reinterpret_cast<const float4*>(pslot) + (gam - g0) * L_eff * 32 + lane;
          const uint32_t* ixp = reinterpret_cast<const uint32_t*>(pslot + p_cs_bytes) + (gam - g0) * L_eff * 32 + lane;
#pragma unroll
          for (int t = 0; t < 8; ++t)
            if (t < L_eff) {
              csr[t] = csp[t * 32];
              ixr[t] = ixp[t * 32];
            }
        } else {
          const int64_t rec = static_cast<int64_t>(gam) * L * 32 + lane;
#pragma unroll
          for (int t = 0; t < 8; ++t)
            if (t < L_eff) {
              csr[t] = __ldg(reinterpret_cast<const float4*>(d.rot_cs) + rec + t * 32);
              ixr[t] = __ldg(reinterpret_cast<const uint32_t*>(d.rot_idx) + rec + t * 32);
            }
        }
      }
      if (have) {
        // two explicit paths: a runtime-selected shared/global pointer would compile to
        // generic loads, which queue behind the weight stream
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int k = (gam - g0) * GRP + lane + 32 * i;
          if (!a.rotate)
            sv[i] = 1.f;
          else if (pstaged && L_eff > 0)
            sv[i] = reinterpret_cast<const float*>(pslot + p_cs_bytes + p_ix_bytes)[k];
          else
            sv[i] = __ldg(d.svec + g0 * GRP + k);
        }
      }
      if (!have) break;
      const int kg = gam * GRP;
#pragma unroll
      for (int b = 0; b < BT; ++b)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int k = lane + 32 * i;
          float v = 0.f;
          if (b < a.B) v = load_act(xs + static_cast<size_t>(b) * x_row_bytes, a.x_bf16, kg - g0 * GRP + k);
          scr[b * 132 + k] = v * sv[i];  // diag(s) x  (a4)
        }
      __syncwarp();
      if (threadIdx.x == 0 && gam == g0) PARO_TL(a, 8);
#pragma unroll
      for (int t = 0; t < 8; ++t) {  // a5: rotations t = 1..L, Eq. 4 form, pre-update values
        if (t >= L_eff) break;
#pragma unroll
        for (int b = 0; b < BT; ++b) {
          float* sb = scr + b * 132;
          const uint32_t i0 = ixr[t] & 0xff, j0 = (ixr[t] >> 8) & 0xff;
          const uint32_t i1 = (ixr[t] >> 16) & 0xff, j1 = ixr[t] >> 24;
          const float a0 = sb[i0], b0 = sb[j0];
          const float a1 = sb[i1], b1 = sb[j1];
          sb[i0] = csr[t].x * a0 - csr[t].y * b0;
          sb[j0] = csr[t].y * a0 + csr[t].x * b0;
          sb[i1] = csr[t].z * a1 - csr[t].w * b1;
          sb[j1] = csr[t].w * a1 + csr[t].z * b1;
        }
        __syncwarp();
        if (threadIdx.x == 0 && gam == g0 && t == 0) PARO_TL(a, 9);
      }
      if (threadIdx.x == 0 && gam == g0) PARO_TL(a, 6);
#pragma unroll
      for (int b = 0; b < BT; ++b) {
        const float* sb = scr + b * 132;
        // perm8 order: pairs (c0, c0+4), (c0+1, c0+5) of the lane's 8-block half
        const uint32_t p0 = pack_half2(sb[c0], sb[c0 + 4]);
        const uint32_t p1 = pack_half2(sb[c0 + 1], sb[c0 + 5]);
        // 32-channel chunk sums of the fp16-rounded x' (chunk = 8 lanes)
        float cs = half2_sum(p0) + half2_sum(p1);
        cs += __shfl_xor_sync(0xffffffffu, cs, 1);
        cs += __shfl_xor_sync(0xffffffffu, cs, 2);
        cs += __shfl_xor_sync(0xffffffffu, cs, 4);
        cs *= TWO_M24;
        const uint32_t uo = u_addr + static_cast<uint32_t>((b * K + kg + b8) * 2 + hh * 8);
        const uint32_t so = s_addr + static_cast<uint32_t>((b * NCH + (kg >> 5) + (lane >> 3)) * 4);
        if (CL > 1) {
          for (uint32_t r = 0; r < CL; ++r) {
            const uint32_t rb = mapa(bar_addr, r);
            st_async_v2(mapa(uo, r), p0, p1, rb);
            if ((lane & 7) == 0) st_async_b32(mapa(so, r), __float_as_uint(cs), rb);
          }
        } else {
          *reinterpret_cast<uint2*>(reinterpret_cast<uint8_t*>(u16) + (uo - u_addr)) = make_uint2(p0, p1);
          if ((lane & 7) == 0) usum[b * NCH + (kg >> 5) + (lane >> 3)] = cs;
        }
      }
      __syncwarp();
      if (threadIdx.x == 0 && gam == g0) PARO_TL(a, 7);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(pfree);  // this warp no longer reads the staged parameters
    if (CL > 1) {
      mbar_wait(xpbar, 0);  // every group's x' has arrived from its owner CTA
    } else {
      named_bar_sync(1, n_compute_warps * 32);
    }
  }
  if (threadIdx.x == 0) PARO_TL(a, 2);

  // ------------------------------------------------------------ phase 2: GEMV
  // warp wk: K slice [wk*512*J, (wk+1)*512*J); lane hl of a half-warp owns 32*J
  // contiguous K (one 128-group).  Slot j of a lane holds chunk (j + hl) % J of its
  // span, so the per-slot 16-byte code loads of the 16 lanes hit distinct banks.
  // row group rg consumes stages rg, rg + RG, ... (all eight row pairs of each)
  const int wk = warp % WK;
  const int rg = warp / WK;
  const int RGN = a.RG;
  const int h = lane >> 4;
  const int hl = lane & 15;
  const int kbase = wk * (512 * J) + hl * (32 * J);
  const bool act = kbase < K;
  uint32_t uP[J][BT][16];
  float Us[BT];
#pragma unroll
  for (int b = 0; b < BT; ++b) {
    Us[b] = 0.f;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int k0 = kbase + 32 * ((j + hl) & (J - 1));
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        uint4 q = make_uint4(0u, 0u, 0u, 0u);
        if (act) q = *reinterpret_cast<const uint4*>(u16 + static_cast<int64_t>(b) * K + k0 + 8 * m);
        uP[j][b][4 * m + 0] = q.x;
        uP[j][b][4 * m + 1] = q.y;
        uP[j][b][4 * m + 2] = q.z;
        uP[j][b][4 * m + 3] = q.w;
      }
      if (act) Us[b] += usum[b * NCH + (k0 >> 5)];
    }
  }
  // inactive lanes (K not a multiple of 512*J) read a valid chunk and contribute 0 (u' = 0)
  const int kb = act ? kbase : 0;
  const int gam = kb >> 7;
  const uint32_t code_off = static_cast<uint32_t>(kb >> 1);
  const int zsh = (gam & 1) * 4;

  // stage slots as 32-bit shared addresses (no generic->shared conversion in the loop)
  const uint32_t ring_a = smem_u32(ring);
  // row group rg owns slots rg, rg + RG, ... so every slot is consumed by one row group
  // in order (mbarrier parity waits can only look one phase ahead)
  const int SP = a.S / RGN;
  for (int st = rg; st < n_stages; st += RGN) {
    const int use = st / RGN;
    const int slot = rg + RGN * (use % SP);
    const uint32_t phase = (use / SP) & 1;
    if (st == n_stages - 1 && threadIdx.x == 0) PARO_TL(a, 10);  // consumer reached the last stage
    mbar_wait(&full[slot], phase);
    if (st == 0 && threadIdx.x == 0) PARO_TL(a, 3);
    if (st == n_stages - 1 && threadIdx.x == 0) PARO_TL(a, 11);  // last stage's bytes landed
    const uint32_t sbase = ring_a + static_cast<uint32_t>(slot) * a.slot_bytes;
    const int r0 = row_begin + st * SR;
    const int nr = min(SR, n_rows - st * SR);
    const uint32_t s_lo = static_cast<uint32_t>((static_cast<int64_t>(r0) * 2 * G) & ~int64_t(15));
    const uint32_t z_lo = static_cast<uint32_t>((static_cast<int64_t>(r0) * ZB) & ~int64_t(15));
    // this lane's row lr = 2i + h: scale, zero and codes addresses (all rows of the slot
    // exist in shared memory; rows past nr hold stale bytes -- computed, never stored)
    const uint32_t sc_a = sbase + a.sc_off + static_cast<uint32_t>(r0 * 2 * G) - s_lo + 2 * gam + h * 2 * G;
    const uint32_t z_a = sbase + a.z_off + static_cast<uint32_t>(r0 * ZB) - z_lo + (gam >> 1) + h * ZB;
    const uint32_t c_a = sbase + code_off + h * (K / 2);
    float racc[RP][BT];
#pragma unroll
    for (int i = 0; i < RP; ++i) {
      const uint32_t row_off = 2 * i;
      uint4 c[J];
#pragma unroll
      for (int j = 0; j < J; ++j) c[j] = lds128_a(c_a + row_off * (K / 2) + 16 * ((j + hl) & (J - 1)));
      const float S = __half2float(__ushort_as_half(lds_u16_a(sc_a + row_off * 2 * G)));
      const float zf = static_cast<float>((lds_u8_a(z_a + row_off * ZB) >> zsh) & 15u);
#pragma unroll
      for (int b = 0; b < BT; ++b) {
        float tl = 0.f, th = 0.f;  // 2^-24 sum q x' over the lane's 32*J codes
#pragma unroll
        for (int j = 0; j < J; ++j) {
          dot_word(c[j].x, &uP[j][b][0], tl, th);
          dot_word(c[j].y, &uP[j][b][4], tl, th);
          dot_word(c[j].z, &uP[j][b][8], tl, th);
          dot_word(c[j].w, &uP[j][b][12], tl, th);
        }
        const float dot = fmaf(0.0625f, th, tl);
        racc[i][b] = S * fmaf(-zf, Us[b], dot);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);  // codes of this stage consumed
    // transpose-reduce the RP row-pair slots across the 16 lanes of each half-warp
#pragma unroll
    for (int b = 0; b < BT; ++b) {
      float v[RP];
#pragma unroll
      for (int i = 0; i < RP; ++i) v[i] = racc[i][b];
      int si = 0;
#pragma unroll
      for (int off = 8, n = RP; off >= 1; off >>= 1) {
        const bool up = hl & off;
        if (n > 1) {
          const int hn = n / 2;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            if (i < hn) {
              const float keep = up ? v[i + hn] : v[i];
              const float send = up ? v[i] : v[i + hn];
              v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
            }
          }
          si = 2 * si + (up ? 1 : 0);
          n = hn;
        } else {
          v[0] += __shfl_xor_sync(0xffffffffu, v[0], off);
        }
      }
      // lanes whose unused low bits are 0 hold slot si (0 <= si < RP)
      const int lr = 2 * si + h;
      const bool writer = (hl & (16 / RP - 1)) == 0;
      if (writer && lr < nr) part[(static_cast<size_t>(wk) * a.rows_max + st * SR + lr) * BT + b] = v[0];
    }
  }
  if (threadIdx.x == 0) PARO_TL(a, 4);
  if (a.pdl) pdl_wait();  // y may still be read by the previous kernel (no-op once it has finished)

  // ------------------------------------------------------------ cross-warp reduction + epilogue (a8)
  named_bar_sync(1, n_compute_warps * 32);
  for (int idx = threadIdx.x; idx < n_rows * BT; idx += n_compute_warps * 32) {
    const int row = idx / BT, b = idx % BT;
    if (b >= a.B) continue;
    float sum = 0.f;
    for (int w = 0; w < WK; ++w) sum += part[(static_cast<size_t>(w) * a.rows_max + row) * BT + b];
    const int64_t n = static_cast<int64_t>(row_begin) + row;
    float v = sum * TWO_P24;
    if (d.bias) v += __ldg(d.bias + n);
    store_out(d.y, a.y_dtype, static_cast<int64_t>(b) * d.N + n, v);
  }
  if (threadIdx.x == 0) PARO_TL(a, 5);
}

// debug: copy the per-CTA event timeline (ns, %globaltimer) of the last debug launch
extern "C" int paro_debug_read_timeline(unsigned long long* host, int n) {
  if (n > 1024 * TL_EVENTS) n = 1024 * TL_EVENTS;
  return static_cast<int>(cudaMemcpyFromSymbol(host, g_paro_timeline, sizeof(unsigned long long) * n));
}

// ============================================================================ host side
int device_sm_count() {
  static int sms = 0;
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  });
  return sms;
}

static int smem_optin() {
  static int v = 0;
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (v <= 0) v = 227 * 1024;
  });
  return v;
}

static inline uint32_t align_up(uint32_t v, uint32_t a) { return (v + a - 1) / a * a; }


static const void* kernel_for(int BT, int J, int big) {
#define PARO_K(BT_, J_, T_) \
  if (BT == BT_ && J == J_ && (big ? 544 : 288) == T_) return reinterpret_cast<const void*>(&paro_gemv_kernel<BT_, J_, T_>);
  PARO_K(1, 1, 288)
  PARO_K(1, 2, 288)
  PARO_K(1, 4, 288)
  PARO_K(2, 1, 288)
  PARO_K(2, 2, 288)
  PARO_K(4, 1, 288)
  PARO_K(1, 1, 544)
  PARO_K(1, 2, 544)
  PARO_K(1, 4, 544)
#undef PARO_K
  return nullptr;
}

// Co-resident CTAs for this launch shape (whole clusters), from the occupancy API.
static int max_resident_ctas(int BT, int J, int threads, int smem, int CL) {
  const void* k = kernel_for(BT, J, threads > 288);
  if (!k) return 0;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) {
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

bool plan_gemv(int B_tile, int n_lin, const int64_t* Ns, const int* Ls, int64_t K, int rotate, GemvConfig* cfg,
               const char** why) {
  GemvConfig c{};
  if (n_lin < 1 || n_lin > GEMV_MAX_LIN) {
    *why = "1..4 linears per decode launch";
    return false;
  }
  int64_t N = 0;
  int L = 0;
  for (int i = 0; i < n_lin; ++i) {
    N += Ns[i];
    L = std::max(L, Ls[i]);
  }
  c.BT = B_tile <= 1 ? 1 : B_tile <= 2 ? 2 : 4;
  const int G = static_cast<int>(K / GRP);
  // J: contiguous 32-K chunks per lane per row (all in one 128-group).  Smallest J that
  // keeps the K slices within 8 warps with <= 6% idle lanes (u' registers: BT * J <= 4);
  // very large K uses up to 16 warps (J = 4).
  int J = 0;
  for (int cand = 1; cand <= 4 && !J; cand *= 2) {
    if (c.BT * cand > 4) break;
    const int64_t span = 512 * cand;
    const int64_t wk = (K + span - 1) / span;
    if (wk <= 8 && (wk * span * 100 <= K * 106 || cand == 4 || K <= span)) J = cand;
  }
  if (!J) J = (c.BT == 1) ? 4 : (c.BT == 2 ? 2 : 1);
  const int WK = static_cast<int>((K + 512 * J - 1) / (512 * J));
  if (WK > 16 || (WK > 8 && c.BT > 1)) {
    *why = "K too large for the decode kernel at this token tile";
    return false;
  }
  // row groups (stage-interleaved): fill up to 8 compute warps per CTA with 2 CTAs/SM,
  // or 16 with 1 CTA/SM
  int ctas_per_sm_pref = 2;
  if (const char* e = getenv("PARO_CTAS_PER_SM")) ctas_per_sm_pref = atoi(e) == 1 ? 1 : 2;
  const int warp_cap = (ctas_per_sm_pref == 1 && c.BT == 1) ? 16 : 8;  // 544-thread variants are BT = 1
  int RG = 1;
  while (RG < 4 && WK * RG * 2 <= warp_cap) RG *= 2;
  if (const char* e = getenv("PARO_RG")) RG = std::max(1, std::min(4, atoi(e)));
  if (WK * RG > 16) RG = 1;
  c.J = J;
  const int sms = device_sm_count();
  const int threads = (WK * RG + 1) * 32;
  // cluster size: share the transform across CTAs (each CTA rotates G/CL groups)
  // (the rotation-off baseline uses the same split, so it differs only by the rotation)
  int CL = 8;
  if (const char* e = getenv("PARO_CLUSTER")) CL = atoi(e);
  if (CL != 1 && CL != 2 && CL != 4 && CL != 8) CL = 8;
  while (CL > 1 && CL > G) CL /= 2;
  c.CL = CL;
  GemvArgs& a = c.a;
  a.n_lin = n_lin;
  a.K = static_cast<int>(K);
  a.G = G;
  a.rotate = rotate;
  a.WK = WK;
  a.RG = RG;
  const int row_bytes = static_cast<int>(K / 2);
  // rows per stage: 2 * RP_PER_STAGE / J (16 rows of <= 2 KB, 4 rows of <= 8 KB, ...)
  const int SR = 2 * RP_PER_STAGE / J;
  a.SR = SR;
  const int ZB = (G + 1) / 2;
  a.sc_off = align_up(static_cast<uint32_t>(SR) * row_bytes, 128);
  a.z_off = a.sc_off + align_up(static_cast<uint32_t>(SR) * 2 * G + 32, 128);
  a.slot_bytes = a.z_off + align_up(static_cast<uint32_t>(SR) * ZB + 32, 128);
  const uint32_t u_bytes = align_up(static_cast<uint32_t>(c.BT) * K * 2, 128);
  const uint32_t usum_bytes = align_up(static_cast<uint32_t>(c.BT) * (K / 32) * 4, 128);
  const int g_per = (G + CL - 1) / CL;
  const uint32_t x_bytes = align_up(static_cast<uint32_t>(c.BT) * g_per * GRP * 2, 128);
  const uint32_t scr_bytes = align_up(static_cast<uint32_t>(WK * RG) * c.BT * 132 * 4, 128);
  // two CTAs per SM when the activation buffer is small (lets the next kernel's weight
  // prefetch start while this one drains, and doubles the warps hiding latency)
  int ctas_per_sm = (u_bytes <= 40 * 1024) ? ctas_per_sm_pref : 1;
  const int budget = (smem_optin() + 1024) / ctas_per_sm - 2048;
  // split the grid's clusters over the linears in proportion to their rows (>= 1 each)
  auto split = [&](int grid) -> bool {
    const int ncl = grid / CL;
    if (ncl < n_lin) return false;
    int cl[GEMV_MAX_LIN], used = 0, big = 0;
    for (int i = 0; i < n_lin; ++i) {
      cl[i] = std::max<int>(1, static_cast<int>(static_cast<double>(ncl) * Ns[i] / N));
      used += cl[i];
      if (Ns[i] > Ns[big]) big = i;
    }
    cl[big] += ncl - used;
    if (cl[big] < 1) return false;
    int begin = 0;
    a.rows_max = 0;
    for (int i = 0; i < n_lin; ++i) {
      GemvLinear& d = a.lin[i];
      d.N = static_cast<int>(Ns[i]);
      d.L = Ls[i];
      d.cta_begin = begin;
      d.n_ctas = cl[i] * CL;
      if (d.n_ctas > Ns[i]) return false;  // at least one row per CTA
      d.rows_base = static_cast<int>(Ns[i] / d.n_ctas);
      d.rows_extra = static_cast<int>(Ns[i] % d.n_ctas);
      a.rows_max = std::max(a.rows_max, d.rows_base + (d.rows_extra ? 1 : 0));
      begin += d.n_ctas;
    }
    return true;
  };
  auto layout = [&](int grid) -> bool {
    if (!split(grid)) return false;
    uint32_t off = 0;
    a.off_u = off;
    off += u_bytes;
    a.off_usum = off;
    off += usum_bytes;
    a.off_x = off;
    off += x_bytes;
    a.off_scr = off;
    off += scr_bytes;
    a.off_part = off;
    off += align_up(static_cast<uint32_t>(WK) * a.rows_max * c.BT * 4, 128);
    a.off_bar = off;
    off += 64 * 16;  // up to 60 stages x (full, empty) + 4 singles
    a.off_ring = align_up(off, 1024);
    const int64_t ring_avail = static_cast<int64_t>(budget) - a.off_ring;
    int S = static_cast<int>(ring_avail / a.slot_bytes);
    const int stages_needed = std::max((a.rows_max + SR - 1) / SR, RG);
    if (S > stages_needed) S = stages_needed;
    if (S > 60) S = 60;
    S -= S % RG;  // each row group owns S / RG slots
    if (S < RG) return false;
    a.S = S;
    a.smem_total = a.off_ring + static_cast<uint32_t>(S) * a.slot_bytes;
    // stage the rotation parameters of this CTA's groups in shared memory: a dedicated
    // region when it fits, else lend the last ring slots (refilled after phase 1)
    a.param_slots = 0;
    a.off_param = 0;
    if (rotate && L > 0) {
      const uint32_t pbytes = static_cast<uint32_t>(g_per) * 32 * L * 20 + static_cast<uint32_t>(g_per) * GRP * 4;
      const int P = static_cast<int>((pbytes + a.slot_bytes - 1) / a.slot_bytes);
      if (static_cast<int64_t>(a.smem_total) + align_up(pbytes, 128) <= budget) {
        a.param_slots = -1;
        a.off_param = a.smem_total;
        a.smem_total += align_up(pbytes, 128);
      } else if (P < S) {
        a.param_slots = P;
      }
    }
    return true;
  };
  int64_t max_ctas = 0;  // at least one row pair per CTA
  for (int i = 0; i < n_lin; ++i) max_ctas += std::max<int64_t>(CL, (Ns[i] + 1) / 2 / CL * CL);
  int grid = sms * ctas_per_sm;
  for (int iter = 0; iter < 3; ++iter) {
    grid = static_cast<int>(std::min<int64_t>(grid, max_ctas)) / CL * CL;
    if (grid < CL * n_lin) grid = CL * n_lin;
    if (!layout(grid)) {
      *why = "decode kernel shared-memory plan does not fit";
      return false;
    }
    const int resident = max_resident_ctas(c.BT, J, threads, static_cast<int>(a.smem_total), CL);
    if (resident <= 0 || resident >= grid) break;
    grid = resident;  // never launch more than one wave
  }
  c.grid = grid;
  if (!layout(grid)) {
    *why = "decode kernel shared-memory plan does not fit";
    return false;
  }
  *cfg = c;
  return true;
}

template <int BT, int J, int T>
static cudaError_t launch_t(const GemvConfig& c, cudaStream_t st) {
  auto kern = paro_gemv_kernel<BT, J, T>;
  static int configured_smem = 0;  // per instantiation
  if (static_cast<int>(c.a.smem_total) > configured_smem) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(c.a.smem_total));
    if (e != cudaSuccess) return e;
    configured_smem = static_cast<int>(c.a.smem_total);
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(c.grid);
  cfg.blockDim = dim3((c.a.WK * c.a.RG + 1) * 32);
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
  const bool big = (c.a.WK * c.a.RG + 1) * 32 > 288;
#define PARO_GEMV_CASE(BT_, J_, T_) \
  if (c.BT == BT_ && c.J == J_ && (big ? 544 : 288) == T_) return launch_t<BT_, J_, T_>(c, st);
  PARO_GEMV_CASE(1, 1, 288)
  PARO_GEMV_CASE(1, 2, 288)
  PARO_GEMV_CASE(1, 4, 288)
  PARO_GEMV_CASE(2, 1, 288)
  PARO_GEMV_CASE(2, 2, 288)
  PARO_GEMV_CASE(4, 1, 288)
  PARO_GEMV_CASE(1, 1, 544)
  PARO_GEMV_CASE(1, 2, 544)
  PARO_GEMV_CASE(1, 4, 544)
#undef PARO_GEMV_CASE
  return cudaErrorInvalidConfiguration;
}

}  // namespace paro
