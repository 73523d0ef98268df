// tile_layout.cuh -- the packed weight layout shared by paro_pack, the decode GEMV, the
// prefill GEMM and the logical unpack (private to the kernels; include/paro.h documents it).
//
// A tile is 32 output rows x one 128-channel group (4096 weights).  Tiles are stored
// row-block-major: tile T = (n / 32) * G + gamma, so the tiles of a run of row blocks are
// one contiguous range in all three arrays.
//   codes : 2048 B per tile.  Row r (0..31) of the tile is 64 bytes at r * 64, read as
//           4 quads t (16 B) x 4 words j (4 B).  Nibble n (bits [4n, 4n+4)) of word (t, j)
//           holds in-group channel tile_k(t, j, n).  The map is chosen so that one AND mask
//           per 32-bit word yields a ready mma.sync A-fragment register: lane (g, t) of the
//           decode GEMV loads quad t of rows g, g+8, g+16, g+24 (LDS.128 each, 512 B apart);
//           for the 16-row MMA block (g, g+8), (w & 0x000F000F) of row g's word j is
//           {A[g][2t], A[g][2t+1]} of MMA 2j as fp16 subnormals q * 2^-24,
//           (w >> 8 & 0x000F000F) is {A[g][2t+8], A[g][2t+9]}, and the 0x00F000F0 masks give
//           the same positions of MMA 2j+1 scaled by 16 (MMA m covers channels 16m..16m+15).
//   scales: 64 B per tile: 32 fp16 S, row r at half index tile_scale_idx(r) (rows g, g+8,
//           g+16, g+24 adjacent: one 64-bit load per lane).
//   zeros : 16 B per tile: 32 uint4 z; the 16-bit word g holds rows g, g+8, g+16, g+24 in
//           nibbles 0..3 (byte tile_zero_byte(r), nibble tile_zero_hi(r)).
// Rows >= N of the last row block are zero in all three arrays.
#pragma once

#ifndef PARO_HD
#define PARO_HD __host__ __device__ __forceinline__
#endif

namespace paro {

constexpr int TILE_ROWS = 32;
constexpr int TILE_CODE_BYTES = 2048;
constexpr int TILE_SCALE_BYTES = 64;
constexpr int TILE_ZERO_BYTES = 16;

// in-group channel held by nibble n of word j of quad t of a tile row
PARO_HD int tile_k(int t, int j, int n) { return 16 * (2 * j + (n & 1)) + 2 * t + ((n >> 2) & 1) + 8 * ((n >> 1) & 1); }

// inverse: channel k (0..127) -> byte within the 64-byte tile row, and nibble (0 low, 1 high)
PARO_HD void tile_pos(int k, int* byte, int* hi) {
  const int m = k >> 4, kk = k & 15;
  const int j = m >> 1, t = (kk & 7) >> 1;
  const int n = (m & 1) | ((kk >> 3) << 1) | ((kk & 1) << 2);
  *byte = t * 16 + j * 4 + (n >> 1);
  *hi = n & 1;
}

PARO_HD int tile_scale_idx(int r) { return 4 * (r & 7) + (r >> 3); }
PARO_HD int tile_zero_byte(int r) { return 2 * (r & 7) + (r >> 4); }
PARO_HD int tile_zero_hi(int r) { return (r >> 3) & 1; }

// Prefill operand order: position (within the group) of the channel held by nibble n of
// word j of quad t, as the prefill dequantiser emits it (32-byte half rows, fp16 pairs
// (n, n+4) per mask).  The prefill pre-stage stores x' in this order.
PARO_HD int prefill_pos(int t, int j, int n) { return 32 * t + 8 * j + 2 * (n & 3) + (n >> 2); }
// channel at prefill position p
PARO_HD int prefill_channel(int p) {
  const int r8 = p & 7;
  return tile_k(p >> 5, (p >> 3) & 3, (r8 >> 1) | ((r8 & 1) << 2));
}

}  // namespace paro
