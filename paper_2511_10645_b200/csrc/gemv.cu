// gemv.cu -- decode path (B <= 8 tokens per launch): scale + L Givens layers fused
// into the activation staging, then the group-wise INT4 dequant GEMV.
//
// SURVEY.md 8(a) rows a4 (stage + scale), a5 (L rotations, Eq. 5 in column form),
// a6 (dequant GEMV), a8 (epilogue).  One kernel:
//
//  * warp `WK*RG` (producer): streams this CTA's contiguous slice of the packed
//    weight (codes / fp16 scales / uint4 zeros, row-major) through a ring of
//    shared-memory stages with cp.async.bulk (TMA engine) + mbarriers.  The first
//    stages are issued before anything else, so the activation transform below
//    runs in the shadow of the first HBM round trip.
//  * compute warps, phase 1 (transform, PAPER.md:195-209's three-level
//    parallelism): the CTAs of a thread-block cluster split the K/128 groups; a
//    warp stages one (group, token) in shared memory, scales by s and applies the
//    L independent rotations (2 pairs per lane per rotation, sync-free inside a
//    rotation, __syncwarp between rotations), then writes the fp16 x' of that
//    group into every CTA of the cluster (DSMEM).  x' never goes to HBM.
//  * compute warps, phase 2 (GEMV): warp (rg, wk) owns a 512*J-wide K slice and
//    every RG-th row pair; half-warp h handles row 2p+h, lane 32 consecutive K.
//    x' lives in registers (fp16 pairs); codes are dequantised in registers with
//    two AND masks per 16-bit half -- a nibble q in bits [0,4) of an fp16 is the
//    subnormal q*2^-24, in bits [4,8) it is 16q*2^-24 -- and multiplied-accumulated
//    with fma.rn.f32.f16 (FHFMA) into fp32: acc = 2^-24 * sum_k q_k x'_k exactly
//    scaled.  Per (row, group): y += S * (acc - z * 2^-24 * sum_k x'_k).
//    Row partials are reduced with a transpose-shuffle over the 16 lanes, then
//    across K-slice warps through shared memory in a fixed order (deterministic).
#include <cstdint>
#include <cstdio>
#include <mutex>

#include "paro_internal.h"
#include "ptx.cuh"

namespace paro {

constexpr int GRP = 128;
constexpr float TWO_M24 = 5.9604644775390625e-08f;  // 2^-24
constexpr float TWO_P24 = 16777216.0f;              // 2^24

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

template <int BT, int J>
struct GemvThreads {  // register budget: u' (16*J*BT) + row accumulators (8*BT) + ~40
  static constexpr int value = (BT * J <= 2) ? 544 : (BT == 1 ? 480 : 288);
};

template <int BT, int J>
__global__ void __launch_bounds__(GemvThreads<BT, J>::value, 1) paro_gemv_kernel(const GemvArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_compute_warps = a.WK * a.RG;
  const bool is_producer = warp == n_compute_warps;
  const int K = a.K, G = a.G, L = a.L;
  const int ZB = (G + 1) >> 1;

  __half* u16 = reinterpret_cast<__half*>(smem + a.off_u);
  float* part = reinterpret_cast<float*>(smem + a.off_part);
  uint8_t* ring = smem + a.off_ring;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.off_bar);
  uint64_t* empty = full + a.S;

  const int cta = blockIdx.x;
  const int n_rows = a.rows_base + (cta < a.rows_extra ? 1 : 0);
  const int row_begin = cta * a.rows_base + min(cta, a.rows_extra);
  const int n_stages = (n_rows + a.SR - 1) / a.SR;
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
    const uint64_t pol = l2_evict_first_policy();
    const int first = min(a.S, n_stages);
    auto issue = [&](int st) {
      const int slot = st % a.S;
      const int r0 = row_begin + st * a.SR;
      const int nr = min(a.SR, n_rows - st * a.SR);
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
    if (lane == 0)
      for (int st = 0; st < first; ++st) issue(st);
    __syncwarp();
    if (a.rotate && CL > 1) {
      cluster_arrive();
      cluster_wait();
    }
    if (lane == 0) {
      for (int st = first; st < n_stages; ++st) {
        const int slot = st % a.S;
        mbar_wait(&empty[slot], ((st / a.S) - 1) & 1);
        issue(st);
      }
    }
    __syncwarp();
    return;
  }

  // ------------------------------------------------------------ phase 1: activation transform
  if (a.pdl) pdl_wait();  // x may be produced by the previous kernel on the stream
  if (a.rotate) {
    float* scr = reinterpret_cast<float*>(smem + a.off_scr) + warp * 132;
    const int my_groups = (G - static_cast<int>(crank) + static_cast<int>(CL) - 1) / static_cast<int>(CL);
    const int items = my_groups * BT;
    for (int it = warp; it < items; it += n_compute_warps) {
      const int gam = static_cast<int>(crank) + (it / BT) * static_cast<int>(CL);
      const int b = it % BT;
      const int kg = gam * GRP;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int k = lane + 32 * i;
        float v = 0.f;
        if (b < a.B) v = load_act(a.x, a.x_bf16, static_cast<int64_t>(b) * K + kg + k) * a.svec[kg + k];
        scr[k] = v;  // diag(s) x  (a4)
      }
      __syncwarp();
      for (int t = 0; t < L; ++t) {  // a5: rotations t = 1..L, Eq. 4 form, pre-update values
        const int64_t e = (static_cast<int64_t>(gam) * L + t) * 64;
        const float2 c0 = a.rot_cs[e + lane], c1 = a.rot_cs[e + lane + 32];
        const uchar2 p0 = a.rot_idx[e + lane], p1 = a.rot_idx[e + lane + 32];
        const float a0 = scr[p0.x], b0 = scr[p0.y];
        const float a1 = scr[p1.x], b1 = scr[p1.y];
        scr[p0.x] = c0.x * a0 - c0.y * b0;
        scr[p0.y] = c0.y * a0 + c0.x * b0;
        scr[p1.x] = c1.x * a1 - c1.y * b1;
        scr[p1.y] = c1.y * a1 + c1.x * b1;
        __syncwarp();
      }
      const uint32_t h01 = pack_half2(scr[4 * lane], scr[4 * lane + 1]);
      const uint32_t h23 = pack_half2(scr[4 * lane + 2], scr[4 * lane + 3]);
      const uint32_t addr = smem_u32(u16 + static_cast<int64_t>(b) * K + kg + 4 * lane);
      for (uint32_t r = 0; r < CL; ++r) {
        const uint32_t ra = (CL > 1) ? mapa(addr, r) : addr;
        if (CL > 1) {
          st_cluster_u32(ra, h01);
          st_cluster_u32(ra + 4, h23);
        } else {
          *reinterpret_cast<uint32_t*>(u16 + static_cast<int64_t>(b) * K + kg + 4 * lane) = h01;
          *reinterpret_cast<uint32_t*>(u16 + static_cast<int64_t>(b) * K + kg + 4 * lane + 2) = h23;
        }
      }
      __syncwarp();
    }
    if (CL > 1) {
      cluster_arrive();
      cluster_wait();
    } else {
      named_bar_sync(1, n_compute_warps * 32);
    }
  }

  // ------------------------------------------------------------ phase 2: GEMV
  const int wk = warp % a.WK;
  const int rg = warp / a.WK;
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
        uint32_t w[4] = {0u, 0u, 0u, 0u};
        if (act[j]) {
          if (a.rotate) {
            const uint4 q = *reinterpret_cast<const uint4*>(u16 + static_cast<int64_t>(b) * K + k0 + 8 * m);
            w[0] = q.x;
            w[1] = q.y;
            w[2] = q.z;
            w[3] = q.w;
          } else if (b < a.B) {
            // rotation disabled (overhead baseline): u = x straight from global
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int64_t base = static_cast<int64_t>(b) * K + k0 + 8 * m + 2 * e;
              w[e] = pack_half2(load_act(a.x, a.x_bf16, base), load_act(a.x, a.x_bf16, base + 1));
            }
          }
        }
        regroup8(w[0], w[1], w[2], w[3], &uP[j][b][4 * m]);
        Us[j][b] += sum8_h(w[0], w[1], w[2], w[3]);
      }
      Us[j][b] *= TWO_M24;  // exact power-of-two scaling
    }
  }

  float racc[8][BT];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int b = 0; b < BT; ++b) racc[i][b] = 0.f;
  int nslot = 0;
  int rp_base = 0;  // CTA-local row-pair index of racc[0]

  auto flush = [&](int count) {
    // transpose-reduce 8 slots across the 16 lanes of this half-warp
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
      const int row = 2 * (rp_base + si * a.RG) + h;  // this warp's slots are every RG-th row pair
      if ((hl & 1) == 0 && si < count && row < n_rows)
        part[(static_cast<size_t>(wk) * a.rows_max + row) * BT + b] = k1;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int b = 0; b < BT; ++b) racc[i][b] = 0.f;
  };

  const int rp_per_stage = a.SR / 2;
  int rp_next = rg;  // next CTA-local row pair this warp owns
  rp_base = rg;
  for (int st = 0; st < n_stages; ++st) {
    const int slot = st % a.S;
    mbar_wait(&full[slot], (st / a.S) & 1);
    const uint8_t* sbase = ring + static_cast<size_t>(slot) * a.slot_bytes;
    const int r0 = row_begin + st * a.SR;
    const int nr = min(a.SR, n_rows - st * a.SR);
    const int64_t s_lo = (static_cast<int64_t>(r0) * 2 * G) & ~int64_t(15);
    const int64_t z_lo = (static_cast<int64_t>(r0) * ZB) & ~int64_t(15);
    const int rp_end = st * rp_per_stage + (nr + 1) / 2;
    for (; rp_next < rp_end; rp_next += a.RG) {
      const int lr = 2 * (rp_next - st * rp_per_stage) + h;  // stage-local row
      const bool valid = lr < nr;
      const uint8_t* crow = sbase + static_cast<size_t>(lr) * (K / 2);
      const int64_t grow = static_cast<int64_t>(r0) + lr;
      float cur[BT];
#pragma unroll
      for (int b = 0; b < BT; ++b) cur[b] = 0.f;
#pragma unroll
      for (int j = 0; j < J; ++j) {
        if (!(act[j] && valid)) continue;
        const int k0 = k0s[j];
        const int gam = k0 >> 7;
        const uint4 c = lds128(crow + (k0 >> 1));
        const float S = __half2float(*reinterpret_cast<const __half*>(sbase + a.sc_off + (grow * 2 * G - s_lo) + 2 * gam));
        const uint8_t zbyte = *(sbase + a.z_off + (grow * ZB - z_lo) + (gam >> 1));
        const float zf = static_cast<float>((zbyte >> ((gam & 1) * 4)) & 15);
#pragma unroll
        for (int b = 0; b < BT; ++b) {
          float acc[4];
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            const uint32_t x = (m == 0) ? c.x : (m == 1) ? c.y : (m == 2) ? c.z : c.w;
            const uint32_t lo = x & 0x000F000Fu, hi = x & 0x00F000F0u;
            const uint32_t x8 = x >> 8;
            const uint32_t lo2 = x8 & 0x000F000Fu, hi2 = x8 & 0x00F000F0u;
            float t = fma_f16lo(lo, uP[j][b][4 * m + 0], 0.f);
            t = fma_f16hi(lo, uP[j][b][4 * m + 0], t);
            t = fma_f16lo(hi, uP[j][b][4 * m + 1], t);
            t = fma_f16hi(hi, uP[j][b][4 * m + 1], t);
            t = fma_f16lo(lo2, uP[j][b][4 * m + 2], t);
            t = fma_f16hi(lo2, uP[j][b][4 * m + 2], t);
            t = fma_f16lo(hi2, uP[j][b][4 * m + 3], t);
            t = fma_f16hi(hi2, uP[j][b][4 * m + 3], t);
            acc[m] = t;
          }
          const float dot = (acc[0] + acc[1]) + (acc[2] + acc[3]);  // = 2^-24 sum q x'
          cur[b] = fmaf(S, fmaf(-zf, Us[j][b], dot), cur[b]);
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int b = 0; b < BT; ++b)
          if (i == nslot) racc[i][b] = cur[b];
      if (++nslot == 8) {
        flush(8);
        nslot = 0;
        rp_base = rp_next + a.RG;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
  }
  if (nslot) flush(nslot);
  if (a.pdl) pdl_launch_dependents();

  // ------------------------------------------------------------ cross-warp reduction + epilogue (a8)
  named_bar_sync(1, n_compute_warps * 32);
  for (int idx = threadIdx.x; idx < n_rows * BT; idx += n_compute_warps * 32) {
    const int row = idx / BT, b = idx % BT;
    if (b >= a.B) continue;
    float sum = 0.f;
    for (int w = 0; w < a.WK; ++w) sum += part[(static_cast<size_t>(w) * a.rows_max + row) * BT + b];
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

bool plan_gemv(int B_tile, int64_t N, int64_t K, int L, int rotate, GemvConfig* cfg, const char** why) {
  GemvConfig c{};
  c.BT = B_tile <= 1 ? 1 : B_tile <= 2 ? 2 : B_tile <= 4 ? 4 : 8;
  const int G = static_cast<int>(K / GRP);
  const int slices = static_cast<int>((K + 511) / 512);
  // J: 32-K chunks per lane per row.  Thread budget per (BT, J) as in GemvThreads.
  auto max_warps = [](int bt, int j) { return ((bt * j <= 2) ? 544 : (bt == 1 ? 480 : 288)) / 32 - 1; };
  int J = 1;
  while ((slices + J - 1) / J > max_warps(c.BT, J) && J < 4) J *= 2;
  const int WK = (slices + J - 1) / J;
  const bool supported = (c.BT == 1) || (c.BT == 2 && J <= 2) || (c.BT == 4 && J == 1);
  if (WK > max_warps(c.BT, J) || !supported) {
    *why = "token tile too wide for this K in the decode kernel";
    return false;
  }
  c.J = J;
  int RG = 1;
  while (RG < 4 && (RG * 2) * WK <= max_warps(c.BT, J) && (RG * 2) * WK <= 16) RG *= 2;
  const int sms = device_sm_count();
  // cluster size: share the transform across CTAs when it is expensive (large K or many tokens)
  int CL = 1;
  if (rotate) {
    const int64_t rot_work = static_cast<int64_t>(K) * c.BT;
    if (rot_work >= 8192) CL = 2;
    if (rot_work >= 16384) CL = 4;
    if (rot_work >= 65536) CL = 8;
    while (CL > 1 && CL > G) CL /= 2;
  }
  c.CL = CL;
  // grid: one CTA per SM (smem-bound), rows split evenly
  int grid = sms;
  grid = grid / CL * CL;
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
  a.RG = RG;
  a.rows_base = static_cast<int>(N / grid);
  a.rows_extra = static_cast<int>(N % grid);
  a.rows_max = a.rows_base + (a.rows_extra ? 1 : 0);
  const int row_bytes = static_cast<int>(K / 2);
  int SR = 8192 / row_bytes;
  SR &= ~1;
  if (SR < 2) SR = 2;
  if (SR > 16) SR = 16;
  a.SR = SR;
  const int ZB = (G + 1) / 2;
  a.sc_off = align_up(static_cast<uint32_t>(SR) * row_bytes, 128);
  a.z_off = a.sc_off + align_up(static_cast<uint32_t>(SR) * 2 * G + 32, 128);
  a.slot_bytes = a.z_off + align_up(static_cast<uint32_t>(SR) * ZB + 32, 128);
  const int nthreads = (WK * RG + 1) * 32;
  uint32_t off = 0;
  a.off_u = off;
  if (rotate) off += align_up(static_cast<uint32_t>(c.BT) * K * 2, 128);
  a.off_scr = off;
  if (rotate) off += align_up(static_cast<uint32_t>(WK * RG) * 132 * 4, 128);
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
  (void)nthreads;
  *cfg = c;
  return true;
}

template <int BT, int J>
static cudaError_t launch_t(const GemvConfig& c, cudaStream_t st) {
  auto kern = paro_gemv_kernel<BT, J>;
  static int configured_smem = 0;  // per instantiation
  if (static_cast<int>(c.a.smem_total) > configured_smem) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin());
    if (e != cudaSuccess) return e;
    configured_smem = smem_optin();
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(c.grid);
  cfg.blockDim = dim3((c.a.WK * c.a.RG + 1) * 32);
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
