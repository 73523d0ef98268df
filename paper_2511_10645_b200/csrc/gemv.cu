// gemv.cu -- decode path (B <= 4 tokens per launch): scale + L Givens layers fused
// into the activation staging, then the group-wise INT4 dequant GEMV.
//
// SURVEY.md 8(a) rows a4 (stage + scale), a5 (L rotations, Eq. 5 in column form),
// a6 (dequant GEMV), a8 (epilogue).  One kernel, launched as clusters of CL CTAs,
// one CTA per SM:
//
//  * producer warp: streams this CTA's contiguous row slice of the packed weight
//    (INT4 codes / fp16 scales / uint4 zeros, row-major) through a ring of
//    shared-memory stages (SR rows each) with cp.async.bulk (TMA engine) +
//    mbarriers.  All stages that fit are issued at kernel start -- before the
//    programmatic-dependent-launch wait -- so the weight stream overlaps both the
//    previous kernel's tail and the activation transform below.
//  * compute warps, phase 1 (transform; PAPER.md:195-209's token / group / pair
//    parallelism): the CL CTAs of a cluster split the K/128 groups; a warp owns a
//    group, keeps its L rotations' (cos, sin, i, j) in registers (loaded before the
//    PDL wait: they do not depend on the previous kernel), stages the group's
//    activations in shared memory, scales by s and applies the L independent
//    rotations (2 pairs per lane per rotation, sync-free inside a rotation,
//    __syncwarp between rotations), then writes fp16 x' into every CTA of the
//    cluster through DSMEM.  x' never goes to HBM.
//  * compute warps, phase 2 (GEMV): warp wk owns a 512*J-wide K slice; half-warp h
//    handles row 2p+h of each row pair, lane 32 consecutive K per chunk.  x' lives
//    in registers as fp16 pairs.  Codes are dequantised in registers with one AND
//    mask per pair of weights: a nibble q in bits [0,4) of an fp16 half IS the
//    subnormal q*2^-24, in bits [4,8) it is 16q*2^-24; fma.rn.f32.f16 (FHFMA)
//    multiplies-accumulates those into fp32, exactly scaled by powers of two.
//    Per (row, group): y += S * (sum q x' - z * sum x').  Row partials are reduced
//    by a transpose-shuffle over the 16 lanes of a half-warp (one per stage of
//    eight row pairs) and across K-slice warps through shared memory in a fixed
//    order (deterministic).
#include <cstdint>
#include <cstdio>
#include <mutex>

#include "paro_internal.h"
#include "ptx.cuh"

namespace paro {

constexpr int GRP = 128;
constexpr float TWO_M24 = 5.9604644775390625e-08f;  // 2^-24
constexpr float TWO_P24 = 16777216.0f;              // 2^24
constexpr int RP_PER_STAGE = 8;                     // max row pairs per stage (SR <= 16 rows)

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

// u32 words w0 = (k0,k1), w1 = (k2,k3), w2 = (k4,k5), w3 = (k6,k7) as fp16 pairs ->
// P[0] = (k0,k4), P[1] = (k1,k5), P[2] = (k2,k6), P[3] = (k3,k7)
__device__ __forceinline__ void regroup8(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, uint32_t* P) {
  P[0] = __byte_perm(w0, w2, 0x5410);
  P[1] = __byte_perm(w0, w2, 0x7632);
  P[2] = __byte_perm(w1, w3, 0x5410);
  P[3] = __byte_perm(w1, w3, 0x7632);
}

__device__ __forceinline__ float sum8_h(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3) {
  float2 a = __half22float2(*reinterpret_cast<__half2*>(&w0));
  float2 b = __half22float2(*reinterpret_cast<__half2*>(&w1));
  float2 c = __half22float2(*reinterpret_cast<__half2*>(&w2));
  float2 d = __half22float2(*reinterpret_cast<__half2*>(&w3));
  return ((a.x + a.y) + (b.x + b.y)) + ((c.x + c.y) + (d.x + d.y));
}

// 2^-24 * sum_{32 k} q_k u_k for one 16-byte chunk of codes (4 words of 8 nibbles).
// Low nibbles carry q*2^-24, high nibbles 16q*2^-24: two kinds of FHFMA chains, the
// high ones scaled by 1/16 at the end (exact).
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

__device__ __forceinline__ float dot32(const uint4 c, const uint32_t* P) {
  float tl0 = 0.f, tl1 = 0.f, th0 = 0.f, th1 = 0.f;
  dot_word(c.x, P + 0, tl0, th0);
  dot_word(c.y, P + 4, tl1, th1);
  dot_word(c.z, P + 8, tl0, th0);
  dot_word(c.w, P + 12, tl1, th1);
  return fmaf(0.0625f, th0 + th1, tl0 + tl1);
}

template <int BT, int J>
struct GemvThreads {  // register budget: u' (16*J*BT) + row accumulators (8*BT) + ~48
  static constexpr int value = (BT * J <= 2) ? 544 : 288;
};

template <int BT, int J>
__global__ void __launch_bounds__(GemvThreads<BT, J>::value, 1) paro_gemv_kernel(const GemvArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int WK = a.WK;
  const int n_compute_warps = WK;
  const bool is_producer = warp == n_compute_warps;
  const int K = a.K, G = a.G, L = a.L;
  const int ZB = (G + 1) >> 1;
  const int SR = a.SR;

  __half* u16 = reinterpret_cast<__half*>(smem + a.off_u);
  float* part = reinterpret_cast<float*>(smem + a.off_part);
  uint8_t* ring = smem + a.off_ring;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.off_bar);
  uint64_t* empty = full + a.S;

  const int cta = blockIdx.x;
  const int n_rows = a.rows_base + (cta < a.rows_extra ? 1 : 0);
  const int row_begin = cta * a.rows_base + min(cta, a.rows_extra);
  const int n_stages = (n_rows + SR - 1) / SR;
  const uint32_t CL = cluster_nctarank();
  const uint32_t crank = cluster_ctarank();

  if (threadIdx.x == 0) {
    for (int i = 0; i < a.S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], n_compute_warps);
    }
    fence_mbar_init();
  }
  if (CL > 1) {
    cluster_arrive();
    cluster_wait();  // mbarriers initialised; every CTA of the cluster is running (DSMEM legal)
  } else {
    __syncthreads();
  }

  // ------------------------------------------------------------ producer warp
  if (is_producer) {
    // Stages [0, S) need no slot release; issue them, then take part in the cluster
    // barrier that publishes x' (the consumers block on it before releasing any slot),
    // then stream the rest of the slice.
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
      bulk_g2s(dst, a.codes + static_cast<int64_t>(r0) * (K / 2), cb, &full[slot], pol);
      bulk_g2s(dst + a.sc_off, a.scales + s_lo, sb, &full[slot], pol);
      bulk_g2s(dst + a.z_off, a.zeros + z_lo, zb, &full[slot], pol);
    };
    const int first = min(a.S, n_stages);
    if (lane == 0)
      for (int st = 0; st < first; ++st) issue(st, st);
    __syncwarp();
    if (a.rotate && CL > 1) {
      cluster_arrive();
      cluster_wait();
    }
    if (lane == 0) {
      int slot = 0;
      uint32_t phase = 1;  // stages >= S: the ring has wrapped once
      for (int st = first; st < n_stages; ++st) {
        mbar_wait(&empty[slot], phase ^ 1);  // stage st - S released by all consumers
        issue(st, slot);
        if (++slot == a.S) {
          slot = 0;
          phase ^= 1;
        }
      }
    }
    __syncwarp();
    return;
  }

  // ------------------------------------------------------------ phase 1: activation transform
  if (a.rotate) {
    float* scr = reinterpret_cast<float*>(smem + a.off_scr) + warp * (BT * 132);
    const int g_per = (G + static_cast<int>(CL) - 1) / static_cast<int>(CL);
    const int g0 = static_cast<int>(crank) * g_per;
    const int g1 = min(G, g0 + g_per);
    bool first = true;
    for (int gam = g0 + warp; gam < g1; gam += n_compute_warps) {
      // rotation parameters of this group -> registers (independent of the previous kernel)
      float2 cs0[8], cs1[8];
      uchar2 ix0[8], ix1[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        if (t < L) {
          const int64_t e = (static_cast<int64_t>(gam) * L + t) * 64;
          cs0[t] = a.rot_cs[e + lane];
          cs1[t] = a.rot_cs[e + lane + 32];
          ix0[t] = a.rot_idx[e + lane];
          ix1[t] = a.rot_idx[e + lane + 32];
        }
      }
      float sv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) sv[i] = a.svec[gam * GRP + lane + 32 * i];
      if (first && a.pdl) pdl_wait();  // x is produced by the previous kernel on the stream
      first = false;
      const int kg = gam * GRP;
#pragma unroll
      for (int b = 0; b < BT; ++b)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int k = lane + 32 * i;
          float v = 0.f;
          if (b < a.B) v = load_act(a.x, a.x_bf16, static_cast<int64_t>(b) * K + kg + k);
          scr[b * 132 + k] = v * sv[i];  // diag(s) x  (a4)
        }
      __syncwarp();
#pragma unroll
      for (int t = 0; t < 8; ++t) {  // a5: rotations t = 1..L, Eq. 4 form, pre-update values
        if (t >= L) break;
#pragma unroll
        for (int b = 0; b < BT; ++b) {
          float* sb = scr + b * 132;
          const float a0 = sb[ix0[t].x], b0 = sb[ix0[t].y];
          const float a1 = sb[ix1[t].x], b1 = sb[ix1[t].y];
          sb[ix0[t].x] = cs0[t].x * a0 - cs0[t].y * b0;
          sb[ix0[t].y] = cs0[t].y * a0 + cs0[t].x * b0;
          sb[ix1[t].x] = cs1[t].x * a1 - cs1[t].y * b1;
          sb[ix1[t].y] = cs1[t].y * a1 + cs1[t].x * b1;
        }
        __syncwarp();
      }
#pragma unroll
      for (int b = 0; b < BT; ++b) {
        const float* sb = scr + b * 132;
        const uint32_t h01 = pack_half2(sb[4 * lane], sb[4 * lane + 1]);
        const uint32_t h23 = pack_half2(sb[4 * lane + 2], sb[4 * lane + 3]);
        __half* dstp = u16 + static_cast<int64_t>(b) * K + kg + 4 * lane;
        if (CL > 1) {
          const uint32_t addr = smem_u32(dstp);
          for (uint32_t r = 0; r < CL; ++r) {
            const uint32_t ra = mapa(addr, r);
            st_cluster_u32(ra, h01);
            st_cluster_u32(ra + 4, h23);
          }
        } else {
          *reinterpret_cast<uint2*>(dstp) = make_uint2(h01, h23);
        }
      }
      __syncwarp();
    }
    if (first && a.pdl) pdl_wait();
    if (CL > 1) {
      cluster_arrive();
      cluster_wait();
    } else {
      named_bar_sync(1, n_compute_warps * 32);
    }
  } else if (a.pdl) {
    pdl_wait();
  }

  // ------------------------------------------------------------ phase 2: GEMV
  const int wk = warp;
  const int h = lane >> 4;
  const int hl = lane & 15;
  uint32_t uP[J][BT][16];
  float Us[J][BT];
  int k0s[J];
  bool act[J];
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int k0 = (wk * J + j) * 512 + hl * 32;
    k0s[j] = k0;
    act[j] = k0 < K;
#pragma unroll
    for (int b = 0; b < BT; ++b) {
      Us[j][b] = 0.f;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        uint4 q = make_uint4(0u, 0u, 0u, 0u);
        if (act[j]) {
          if (a.rotate) {
            q = *reinterpret_cast<const uint4*>(u16 + static_cast<int64_t>(b) * K + k0 + 8 * m);
          } else if (b < a.B) {
            // rotation disabled (overhead baseline): u = x straight from global (16-byte loads)
            q = __ldg(reinterpret_cast<const uint4*>(static_cast<const uint8_t*>(a.x) +
                                                     (static_cast<int64_t>(b) * K + k0 + 8 * m) * 2));
            if (a.x_bf16) {
              uint32_t* e = reinterpret_cast<uint32_t*>(&q);
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&e[i]));
                e[i] = pack_half2(f.x, f.y);
              }
            }
          }
        }
        regroup8(q.x, q.y, q.z, q.w, &uP[j][b][4 * m]);
        Us[j][b] += sum8_h(q.x, q.y, q.z, q.w);
      }
      Us[j][b] *= TWO_M24;  // exact power-of-two scaling
    }
  }

  int slot = 0;
  uint32_t phase = 0;
  for (int st = 0; st < n_stages; ++st) {
    mbar_wait(&full[slot], phase);
    const uint8_t* sbase = ring + static_cast<size_t>(slot) * a.slot_bytes;
    const int r0 = row_begin + st * SR;
    const int nr = min(SR, n_rows - st * SR);
    const int64_t s_lo = (static_cast<int64_t>(r0) * 2 * G) & ~int64_t(15);
    const int64_t z_lo = (static_cast<int64_t>(r0) * ZB) & ~int64_t(15);
    const uint8_t* sc_base = sbase + a.sc_off + (static_cast<int64_t>(r0) * 2 * G - s_lo);
    const uint8_t* z_base = sbase + a.z_off + (static_cast<int64_t>(r0) * ZB - z_lo);
    float racc[RP_PER_STAGE][BT];
#pragma unroll
    for (int i = 0; i < RP_PER_STAGE; ++i) {
#pragma unroll
      for (int b = 0; b < BT; ++b) racc[i][b] = 0.f;
      const int lr = 2 * i + h;  // stage-local row
      if (2 * i < SR && lr < nr) {
        const uint8_t* crow = sbase + static_cast<size_t>(lr) * (K / 2);
#pragma unroll
        for (int j = 0; j < J; ++j) {
          if (!act[j]) continue;
          const int k0 = k0s[j];
          const int gam = k0 >> 7;
          const uint4 c = lds128(crow + (k0 >> 1));
          const float S = __half2float(*reinterpret_cast<const __half*>(sc_base + lr * 2 * G + 2 * gam));
          const uint32_t zbyte = *(z_base + lr * ZB + (gam >> 1));
          const float zf = static_cast<float>((zbyte >> ((gam & 1) * 4)) & 15u);
#pragma unroll
          for (int b = 0; b < BT; ++b) {
            const float dot = dot32(c, uP[j][b]);  // = 2^-24 sum q x'
            racc[i][b] = fmaf(S, fmaf(-zf, Us[j][b], dot), racc[i][b]);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);  // codes of this stage consumed
    // transpose-reduce the 8 row-pair slots across the 16 lanes of each half-warp
#pragma unroll
    for (int b = 0; b < BT; ++b) {
      const bool b3 = hl & 8, b2 = hl & 4, b1 = hl & 2;
      float k4[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float keep = b3 ? racc[i + 4][b] : racc[i][b];
        const float send = b3 ? racc[i][b] : racc[i + 4][b];
        k4[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
      }
      float k2[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const float keep = b2 ? k4[i + 2] : k4[i];
        const float send = b2 ? k4[i] : k4[i + 2];
        k2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
      }
      float k1 = (b1 ? k2[1] : k2[0]) + __shfl_xor_sync(0xffffffffu, b1 ? k2[0] : k2[1], 2);
      k1 += __shfl_xor_sync(0xffffffffu, k1, 1);
      const int si = hl >> 1;
      const int lr = 2 * si + h;
      if ((hl & 1) == 0 && lr < nr)
        part[(static_cast<size_t>(wk) * a.rows_max + st * SR + lr) * BT + b] = k1;
    }
    if (++slot == a.S) {
      slot = 0;
      phase ^= 1;
    }
  }
  if (a.pdl) pdl_launch_dependents();

  // ------------------------------------------------------------ cross-warp reduction + epilogue (a8)
  named_bar_sync(1, n_compute_warps * 32);
  for (int idx = threadIdx.x; idx < n_rows * BT; idx += n_compute_warps * 32) {
    const int row = idx / BT, b = idx % BT;
    if (b >= a.B) continue;
    float sum = 0.f;
    for (int w = 0; w < WK; ++w) sum += part[(static_cast<size_t>(w) * a.rows_max + row) * BT + b];
    const int64_t n = static_cast<int64_t>(row_begin) + row;
    float v = sum * TWO_P24;
    if (a.bias) v += a.bias[n];
    store_out(a.y, a.y_dtype, static_cast<int64_t>(b) * a.N + n, v);
  }
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

static int max_compute_warps(int bt, int j) { return ((bt * j <= 2) ? 544 : 288) / 32 - 1; }

bool plan_gemv(int B_tile, int64_t N, int64_t K, int L, int rotate, GemvConfig* cfg, const char** why) {
  GemvConfig c{};
  c.BT = B_tile <= 1 ? 1 : B_tile <= 2 ? 2 : 4;
  const int G = static_cast<int>(K / GRP);
  const int slices = static_cast<int>((K + 511) / 512);
  // J: 32-K chunks per lane per row.  Prefer J=2 once the K-slices need more than 8 warps.
  int J = 1;
  while (J < 4 && ((slices + J - 1) / J > max_compute_warps(c.BT, J) || (slices + J - 1) / J > 8)) J *= 2;
  const int WK = (slices + J - 1) / J;
  const bool supported = (c.BT == 1) || (c.BT == 2 && J <= 2) || (c.BT == 4 && J == 1);
  if (WK > max_compute_warps(c.BT, J) || !supported) {
    *why = "token tile too wide for this K in the decode kernel";
    return false;
  }
  c.J = J;
  const int sms = device_sm_count();
  // cluster size: share the transform across CTAs (each CTA rotates G/CL groups)
  int CL = 1;
  if (rotate) {
    CL = 8;
    while (CL > 1 && CL > G) CL /= 2;
  }
  c.CL = CL;
  // grid: one CTA per SM (shared-memory ring), rows split evenly
  int grid = sms / CL * CL;
  const int64_t max_ctas = (N + 1) / 2;  // at least one row pair per CTA
  if (grid > max_ctas) grid = static_cast<int>(max_ctas) / CL * CL;
  if (grid < CL) grid = CL;
  c.grid = grid;
  GemvArgs& a = c.a;
  a.N = static_cast<int>(N);
  a.K = static_cast<int>(K);
  a.G = G;
  a.L = L;
  a.rotate = rotate;
  a.WK = WK;
  a.RG = 1;
  a.rows_base = static_cast<int>(N / grid);
  a.rows_extra = static_cast<int>(N % grid);
  a.rows_max = a.rows_base + (a.rows_extra ? 1 : 0);
  const int row_bytes = static_cast<int>(K / 2);
  // rows per stage: ~32 KB of codes, even, at most 2 * RP_PER_STAGE
  int SR = 32768 / row_bytes;
  SR &= ~1;
  if (SR < 2) SR = 2;
  if (SR > 2 * RP_PER_STAGE) SR = 2 * RP_PER_STAGE;
  a.SR = SR;
  const int ZB = (G + 1) / 2;
  a.sc_off = align_up(static_cast<uint32_t>(SR) * row_bytes, 128);
  a.z_off = a.sc_off + align_up(static_cast<uint32_t>(SR) * 2 * G + 32, 128);
  a.slot_bytes = a.z_off + align_up(static_cast<uint32_t>(SR) * ZB + 32, 128);
  uint32_t off = 0;
  a.off_u = off;
  if (rotate) off += align_up(static_cast<uint32_t>(c.BT) * K * 2, 128);
  a.off_scr = off;
  if (rotate) off += align_up(static_cast<uint32_t>(WK) * c.BT * 132 * 4, 128);
  a.off_part = off;
  off += align_up(static_cast<uint32_t>(WK) * a.rows_max * c.BT * 4, 128);
  a.off_bar = off;
  off += 64 * 16;  // up to 64 stages x (full, empty)
  a.off_ring = align_up(off, 1024);
  const int budget = smem_optin() - 1024;
  const int64_t ring_avail = static_cast<int64_t>(budget) - a.off_ring;
  int S = static_cast<int>(ring_avail / a.slot_bytes);
  const int stages_needed = (a.rows_max + SR - 1) / SR;
  if (S > stages_needed) S = stages_needed;
  if (S > 64) S = 64;
  if (S < 1) {
    *why = "decode kernel shared-memory plan does not fit";
    return false;
  }
  a.S = S;
  a.smem_total = a.off_ring + static_cast<uint32_t>(S) * a.slot_bytes;
  *cfg = c;
  return true;
}

template <int BT, int J>
static cudaError_t launch_t(const GemvConfig& c, cudaStream_t st) {
  auto kern = paro_gemv_kernel<BT, J>;
  static int configured_smem = 0;  // per instantiation
  if (static_cast<int>(c.a.smem_total) > configured_smem) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(c.a.smem_total));
    if (e != cudaSuccess) return e;
    configured_smem = static_cast<int>(c.a.smem_total);
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(c.grid);
  cfg.blockDim = dim3((c.a.WK + 1) * 32);
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
#define PARO_GEMV_CASE(BT_, J_) \
  if (c.BT == BT_ && c.J == J_) return launch_t<BT_, J_>(c, st);
  PARO_GEMV_CASE(1, 1)
  PARO_GEMV_CASE(1, 2)
  PARO_GEMV_CASE(1, 4)
  PARO_GEMV_CASE(2, 1)
  PARO_GEMV_CASE(2, 2)
  PARO_GEMV_CASE(4, 1)
#undef PARO_GEMV_CASE
  return cudaErrorInvalidConfiguration;
}

}  // namespace paro
