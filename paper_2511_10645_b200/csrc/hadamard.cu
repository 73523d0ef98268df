// hadamard.cu -- fast Walsh-Hadamard transform of activations (the comparison transform of the
// paper's kernel experiment, fig:kernel-speedup: "speedup of our transform
// (with 8 independent rotations) over the fast Hadamard transform ... increases with the channel
// dimension, because the Hadamard transform has inherent dependencies across all channels").
// SURVEY.md 8(f) NEXT #2; SPEC.md:336-344 (fwht: unnormalised butterfly; the randomised variant
// applies signs, then the butterfly, then scales).
//
// y = scale * H_n diag(signs) x per token, n = 2^k (256 .. 16384), H_n the Sylvester Hadamard
// matrix (H[i, j] = (-1)^popcount(i & j)), so H_n = H_R (x) H_C for any split of the index bits
// and the butterfly stages on different bits commute.  fp32 arithmetic, fp16 output.
// One token = n / 16 threads; every thread holds 16 values in registers:
//  * phase A: 16 CONTIGUOUS elements (two 16-byte loads): stages on index bits 0-3 in registers,
//    bits 4-8 by warp shuffles (xor over lane bits: partner lanes hold the partner elements);
//  * phase B (n > 512): the token goes through shared memory once (a transpose); the thread now
//    holds elements c + 512 m of column c, and the stages on bits >= 9 run in registers (and,
//    for n = 16384, one more shuffle between the two threads sharing a column); stores go out
//    from this layout (consecutive threads = consecutive columns: coalesced).
// Bound: HBM (2n bytes in + 2n out per token) at large token counts, latency at small ones.
#include <cstdint>

#include "paro_internal.h"
#include "ptx.cuh"

namespace paro {

namespace {

template <int LOGN>
__global__ void __launch_bounds__(LOGN >= 11 ? (1 << (LOGN - 4)) : 128) fwht_kernel(
    const void* __restrict__ x, int x_bf16, int64_t T, const float* __restrict__ signs, float scale,
    __half* __restrict__ y) {
  constexpr int n = 1 << LOGN;
  constexpr int TPR = n / 16;                  // threads per token
  constexpr int RPC = TPR >= 128 ? 1 : 128 / TPR;  // tokens per CTA
  constexpr int SHUF = LOGN - 4 < 5 ? LOGN - 4 : 5;  // shuffle stages of phase A (bits 4 .. 4 + SHUF - 1)
  constexpr int RB = LOGN - 4 - SHUF;          // bits left for phase B (0 when n <= 512)
  extern __shared__ __align__(16) float fsm[];
  const int tr = threadIdx.x % TPR, rr = threadIdx.x / TPR;
  const int64_t tok = static_cast<int64_t>(blockIdx.x) * RPC + rr;
  const bool live = tok < T;
  float v[16];
  // ---- load 16 contiguous elements (and the random signs)
  {
    const int64_t base = tok * n + tr * 16;
    uint4 q0 = make_uint4(0u, 0u, 0u, 0u), q1 = q0;
    if (live) {
      q0 = __ldg(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(x) + base));
      q1 = __ldg(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(x) + base) + 1);
    }
    const uint32_t w[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      float2 f;
      if (x_bf16)
        f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
      else
        f = __half22float2(*reinterpret_cast<const __half2*>(&w[e]));
      v[2 * e] = f.x;
      v[2 * e + 1] = f.y;
    }
    if (signs) {
#pragma unroll
      for (int e = 0; e < 16; e += 4) {
        const float4 sg = __ldg(reinterpret_cast<const float4*>(signs + tr * 16 + e));
        v[e] *= sg.x;
        v[e + 1] *= sg.y;
        v[e + 2] *= sg.z;
        v[e + 3] *= sg.w;
      }
    }
  }
  // ---- phase A: bits 0-3 in registers
#pragma unroll
  for (int h = 1; h < 16; h <<= 1)
#pragma unroll
    for (int e = 0; e < 16; ++e)
      if (!(e & h)) {
        const float a = v[e], b = v[e + h];
        v[e] = a + b;
        v[e + h] = a - b;
      }
  // bits 4 .. 4 + SHUF - 1: the partner of element e of lane l is element e of lane l ^ m
#pragma unroll
  for (int s = 0; s < SHUF; ++s) {
    const int m = 1 << s;
    const bool upper = (tr & m) != 0;
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const float o = __shfl_xor_sync(0xffffffffu, v[e], m);
      v[e] = upper ? o - v[e] : v[e] + o;
    }
  }
  if constexpr (RB == 0) {
    if (live) {
      const int64_t base = tok * n + tr * 16;
      uint32_t w[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const __half2 hv = __floats2half2_rn(v[2 * e] * scale, v[2 * e + 1] * scale);
        w[e] = *reinterpret_cast<const uint32_t*>(&hv);
      }
      reinterpret_cast<uint4*>(y + base)[0] = make_uint4(w[0], w[1], w[2], w[3]);
      reinterpret_cast<uint4*>(y + base)[1] = make_uint4(w[4], w[5], w[6], w[7]);
    }
  } else {
    // ---- phase B: transpose through shared memory; element i = c + 512 m (c < 512, m < 2^RB)
    constexpr int M = 1 << RB;                       // elements per column
    constexpr int CPT = M <= 16 ? 16 / M : 1;        // columns per thread
    constexpr int TPC = M <= 16 ? 1 : M / 16;        // threads per column (n = 16384: 2)
    constexpr int EPC = M / TPC;                     // elements of a column per thread
    // element i at sm[i + i / 32]: the phase-A writes (thread tr: i = 16 tr + e) and the
    // column reads (consecutive threads: consecutive c) are both bank-conflict free
    float* sm = fsm + rr * (n + n / 32);
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int i = tr * 16 + e;
      sm[i + (i >> 5)] = v[e];
    }
    __syncthreads();
    // column ownership: thread tr -> columns c = (tr / TPC) + j * (TPR / TPC), part tr % TPC
    const int part = tr % TPC, c0 = tr / TPC;
    constexpr int CSTRIDE = TPR / TPC;
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
      const int c = c0 + j * CSTRIDE;
#pragma unroll
      for (int e = 0; e < EPC; ++e) {
        const int m = part * EPC + e;
        const int i = c + 512 * m;
        v[j * EPC + e] = sm[i + (i >> 5)];
      }
    }
    // stages on bits 9 .. : in registers within a column (element index m)
#pragma unroll
    for (int j = 0; j < CPT; ++j)
#pragma unroll
      for (int h = 1; h < EPC; h <<= 1)
#pragma unroll
        for (int e = 0; e < EPC; ++e)
          if (!(e & h)) {
            const float a = v[j * EPC + e], b = v[j * EPC + e + h];
            v[j * EPC + e] = a + b;
            v[j * EPC + e + h] = a - b;
          }
    if constexpr (TPC == 2) {  // the top bit: the partner thread of the column (lane ^ 1)
      const bool upper = part != 0;
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const float o = __shfl_xor_sync(0xffffffffu, v[e], 1);
        v[e] = upper ? o - v[e] : v[e] + o;
      }
    }
    if (live) {
#pragma unroll
      for (int j = 0; j < CPT; ++j) {
        const int c = c0 + j * CSTRIDE;
#pragma unroll
        for (int e = 0; e < EPC; ++e) {
          const int m = part * EPC + e;
          y[tok * n + c + 512 * m] = __float2half_rn(v[j * EPC + e] * scale);
        }
      }
    }
  }
}

template <int LOGN>
cudaError_t fwht_launch(const void* x, int x_bf16, int64_t T, const float* signs, float scale, __half* y,
                        cudaStream_t st) {
  constexpr int n = 1 << LOGN, TPR = n / 16, RPC = TPR >= 128 ? 1 : 128 / TPR;
  const int threads = TPR * RPC;
  const int smem = LOGN > 9 ? static_cast<int>(RPC * (n + n / 32) * sizeof(float)) : 0;
  const void* k = reinterpret_cast<const void*>(&fwht_kernel<LOGN>);
  if (smem > 48 * 1024) {
    cudaError_t e = ensure_smem_attr(k, smem);
    if (e != cudaSuccess) return e;
  }
  const int64_t grid = (T + RPC - 1) / RPC;
  fwht_kernel<LOGN><<<static_cast<unsigned>(grid), threads, smem, st>>>(x, x_bf16, T, signs, scale, y);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_fwht(const void* x, int x_bf16, int64_t T, int64_t n, const float* signs, float scale, void* y,
                        cudaStream_t st) {
  __half* yo = static_cast<__half*>(y);
  switch (n) {
    case 256: return fwht_launch<8>(x, x_bf16, T, signs, scale, yo, st);
    case 512: return fwht_launch<9>(x, x_bf16, T, signs, scale, yo, st);
    case 1024: return fwht_launch<10>(x, x_bf16, T, signs, scale, yo, st);
    case 2048: return fwht_launch<11>(x, x_bf16, T, signs, scale, yo, st);
    case 4096: return fwht_launch<12>(x, x_bf16, T, signs, scale, yo, st);
    case 8192: return fwht_launch<13>(x, x_bf16, T, signs, scale, yo, st);
    case 16384: return fwht_launch<14>(x, x_bf16, T, signs, scale, yo, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace paro
