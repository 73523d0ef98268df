// pack.cu -- paro_pack's device part: fold T into W (Eq. 8) and RTN-quantise (Eq. 1).
//
// Offline step.  fp64 throughout with explicitly
// rounded intrinsics (__dmul_rn / __dsub_rn / __dadd_rn / __ddiv_rn) and this TU
// is compiled with -fmad=false, so every product and sum is rounded separately
// (Q7) -- required for bit-exact codes/scales/zeros.
//
// Mapping: one CTA = PACK_ROWS weight rows, looping over the K/128 groups; results are
// written in the tile layout of tile_layout.cuh.
// Thread (r, p), p in [0, 64): holds slot p of the current rotation for row r.
#include <cstdint>
#include <cuda_fp16.h>

#include "paro_internal.h"
#include "tile_layout.cuh"

namespace paro {

constexpr int PACK_ROWS = 4;
constexpr int G_ = 128;

__device__ __forceinline__ uint16_t f64_to_f16_rne_bits(double v) {
  // cvt.rn.f16.f64: a single round-to-nearest-even from fp64 (no double rounding via fp32).
  uint16_t h;
  asm("cvt.rn.f16.f64 %0, %1;" : "=h"(h) : "d"(v));
  return h;
}

__global__ void __launch_bounds__(PACK_ROWS * 64) pack_fold_rtn_kernel(
    const __half* __restrict__ W, const float* __restrict__ s, const double2* __restrict__ cs64,
    const uchar2* __restrict__ idx, int64_t N, int64_t K, int L, uint8_t* __restrict__ codes,
    __half* __restrict__ scales, uint8_t* __restrict__ zeros, int* __restrict__ status) {
  const int G = static_cast<int>(K / G_);
  const int r = threadIdx.x / 64;
  const int p = threadIdx.x % 64;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * PACK_ROWS + r;
  const bool live = row < N;

  __shared__ double v[PACK_ROWS][G_ + 2];
  __shared__ double red_mn[PACK_ROWS][2], red_mx[PACK_ROWS][2];
  __shared__ double Ssh[PACK_ROWS];
  __shared__ double zsh[PACK_ROWS];
  __shared__ uint8_t qsh[PACK_ROWS][G_];
  const int rt = static_cast<int>(row % TILE_ROWS);  // row within its tile

  int bad = 0;
  for (int gam = 0; gam < G; ++gam) {
    // v = diag(alpha) w = w / s  (one correctly-rounded division, Q3)
    for (int h = 0; h < 2; ++h) {
      const int k = p + 64 * h;
      double w = 0.0;
      if (live) w = static_cast<double>(__half2float(W[row * K + static_cast<int64_t>(gam) * G_ + k]));
      const double sv = static_cast<double>(s[gam * G_ + k]);
      v[r][k] = __ddiv_rn(w, sv);
    }
    __syncthreads();
    // t = 1..L independent rotations, Eq. 4, pre-update values.
    for (int t = 0; t < L; ++t) {
      const int64_t e = (static_cast<int64_t>(gam) * L + t) * 64 + p;
      const uchar2 ij = idx[e];
      if (ij.x < G_) {
        const double2 c = cs64[e];
        const double a = v[r][ij.x];
        const double b = v[r][ij.y];
        v[r][ij.x] = __dsub_rn(__dmul_rn(c.x, a), __dmul_rn(c.y, b));
        v[r][ij.y] = __dadd_rn(__dmul_rn(c.y, a), __dmul_rn(c.x, b));
      }
      __syncthreads();
    }
    // Eq. 1 on the 128 folded values of (row, gam): min / max
    const double v0 = v[r][p], v1 = v[r][p + 64];
    double mn = fmin(v0, v1), mx = fmax(v0, v1);
    if (!(isfinite(v0) && isfinite(v1))) bad |= 1;
    for (int o = 16; o > 0; o >>= 1) {
      mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if ((p & 31) == 0) {
      red_mn[r][p >> 5] = mn;
      red_mx[r][p >> 5] = mx;
    }
    __syncthreads();
    if (p == 0) {
      const double gmn = fmin(red_mn[r][0], red_mn[r][1]);
      const double gmx = fmax(red_mx[r][0], red_mx[r][1]);
      const double s64 = __ddiv_rn(__dsub_rn(gmx, gmn), 15.0);
      uint16_t hb = f64_to_f16_rne_bits(s64);
      if ((hb & 0x7fffu) == 0) hb = 0x0001u;  // floor at 2^-24 (Q10); s64 >= 0 so no sign
      if ((hb & 0x7c00u) == 0x7c00u) bad |= 2;  // fp16 overflow (or NaN)
      const double S = static_cast<double>(__half2float(__ushort_as_half(hb)));
      double z = -rint(__ddiv_rn(gmn, S));     // z = -round(min / S), half-even (Q9)
      z = fmin(fmax(z, 0.0), 15.0);              // clamp to [0, 2^b - 1] (Q11)
      Ssh[r] = S;
      zsh[r] = z;
      if (live) {  // tile layout (tile_layout.cuh); buffers were zeroed before the launch
        const int64_t T = (row / TILE_ROWS) * G + gam;
        scales[T * TILE_ROWS + tile_scale_idx(rt)] = __ushort_as_half(hb);
        const int64_t zbyte = T * TILE_ZERO_BYTES + tile_zero_byte(rt);
        atomicOr(reinterpret_cast<unsigned int*>(zeros + (zbyte & ~int64_t(3))),
                 static_cast<unsigned int>(z) << (8 * (zbyte & 3) + 4 * tile_zero_hi(rt)));
      }
    }
    __syncthreads();
    {
      const double S = Ssh[r], z = zsh[r];
      for (int h = 0; h < 2; ++h) {
        const int k = p + 64 * h;
        double q = __dadd_rn(rint(__ddiv_rn(v[r][k], S)), z);
        q = fmin(fmax(q, 0.0), 15.0);
        qsh[r][k] = static_cast<uint8_t>(q);
      }
    }
    __syncthreads();
    if (live) {
      // byte p of the row's 64 code bytes in its tile: quad p / 16, word (p / 4) % 4,
      // nibbles 2 (p % 4) (low) and 2 (p % 4) + 1 (high) -> channels tile_k(...)
      const int tq = p >> 4, wj = (p >> 2) & 3, bw = p & 3;
      const uint8_t b = static_cast<uint8_t>(qsh[r][tile_k(tq, wj, 2 * bw)] | (qsh[r][tile_k(tq, wj, 2 * bw + 1)] << 4));
      const int64_t T = (row / TILE_ROWS) * G + gam;
      codes[T * TILE_CODE_BYTES + rt * 64 + p] = b;
    }
    __syncthreads();
  }
  if (bad) atomicOr(status, bad);
}

cudaError_t launch_pack(const void* W, const float* s, const void* cs64, const void* idx, int64_t N, int64_t K, int L,
                        void* codes, void* scales, void* zeros, int* status, cudaStream_t st) {
  const int G = static_cast<int>(K / G_);
  const unsigned grid = static_cast<unsigned>((N + PACK_ROWS - 1) / PACK_ROWS);
  (void)G;
  pack_fold_rtn_kernel<<<grid, PACK_ROWS * 64, 0, st>>>(
      static_cast<const __half*>(W), s, static_cast<const double2*>(cs64), static_cast<const uchar2*>(idx), N, K, L,
      static_cast<uint8_t*>(codes), static_cast<__half*>(scales), static_cast<uint8_t*>(zeros), status);
  return cudaGetLastError();
}

}  // namespace paro
