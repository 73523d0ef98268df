// pairs.cpp -- paro_select_pairs: Alg. A1 "Selection of Independent Channel Pairs"
// ("skip pairs that have already been selected"), the
// step upstream of paro_pack.  Host code: the algorithm is a
// sequential greedy scan per group and runs once, offline.
//
// Representation (not the paper's g x g matrices): a channel-availability bitmask per
// rotation (A_rot's rows/columns are all-zero exactly for the channels taken in this
// rotation) and one "pair used" flag per lexicographic pair index (A's zeroed entries).
// A_rot[i, j] = 0  <=>  channel i or j taken in this rotation, or (i, j) taken earlier.
//
// Random shuffle (reading Q20): SplitMix64 -> xoshiro256**,
// Fisher-Yates from the last element down with an unbiased bounded draw (reject draws
// below 2^64 mod m).  Group gamma's state = SplitMix64(seed) outputs 4 gamma .. 4 gamma + 3.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <vector>

#include "paro.h"
#include "paro_internal.h"

namespace {

struct SplitMix64 {
  uint64_t x;
  uint64_t next() {
    uint64_t z = (x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
};

struct Xoshiro256ss {
  uint64_t s[4];
  static uint64_t rotl(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }
  uint64_t next() {
    const uint64_t r = rotl(s[1] * 5, 7) * 9, t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return r;
  }
  uint64_t bounded(uint64_t m) {  // uniform in [0, m)
    const uint64_t lim = (0 - m) % m;  // 2^64 mod m
    for (;;) {
      const uint64_t r = next();
      if (r >= lim) return r % m;
    }
  }
};

}  // namespace

extern "C" paro_status paro_select_pairs(int64_t n_groups, int32_t g, int32_t n_rot, int32_t n_pairs, uint64_t seed,
                                         int16_t* pairs_out) {
  if (g < 2 || g > 4096 || n_rot < 1 || n_pairs < 1 || n_pairs > g / 2 || n_groups < 0)
    return static_cast<paro_status>(
        paro::set_error(PARO_ERR_INVALID_ARGUMENT, "paro_select_pairs: need 2 <= g <= 4096, n_rot >= 1, 1 <= n_pairs <= g/2"));
  if (n_groups > 0 && pairs_out == nullptr)
    return static_cast<paro_status>(paro::set_error(PARO_ERR_INVALID_ARGUMENT, "paro_select_pairs: pairs_out is NULL"));
  const uint32_t np = static_cast<uint32_t>(g) * (g - 1) / 2;
  // lexicographic pair index -> (i, j)
  std::vector<uint16_t> pi(np), pj(np);
  for (uint32_t i = 0, k = 0; i < static_cast<uint32_t>(g); ++i)
    for (uint32_t j = i + 1; j < static_cast<uint32_t>(g); ++j, ++k) {
      pi[k] = static_cast<uint16_t>(i);
      pj[k] = static_cast<uint16_t>(j);
    }
  std::vector<uint32_t> perm(np);
  std::vector<uint8_t> used(np);
  std::vector<uint64_t> taken((g + 63) / 64);
  SplitMix64 sm{seed};
  const size_t per_group = static_cast<size_t>(n_rot) * n_pairs * 2;
  for (int64_t gam = 0; gam < n_groups; ++gam) {
    Xoshiro256ss rng;
    for (int w = 0; w < 4; ++w) rng.s[w] = sm.next();  // outputs 4 gam .. 4 gam + 3
    for (uint32_t k = 0; k < np; ++k) perm[k] = k;
    for (uint32_t i = np - 1; i > 0; --i) {
      const uint32_t j = static_cast<uint32_t>(rng.bounded(i + 1ull));
      const uint32_t t = perm[i];
      perm[i] = perm[j];
      perm[j] = t;
    }
    std::memset(used.data(), 0, np);
    int16_t* out = pairs_out + gam * per_group;
    for (size_t e = 0; e < per_group; ++e) out[e] = -1;
    for (int r = 0; r < n_rot; ++r) {
      std::fill(taken.begin(), taken.end(), 0ull);
      int cnt = 0;
      for (uint32_t k = 0; k < np && cnt < n_pairs; ++k) {
        const uint32_t q = perm[k];
        const uint32_t i = pi[q], j = pj[q];
        if (used[q] || ((taken[i >> 6] >> (i & 63)) & 1u) || ((taken[j >> 6] >> (j & 63)) & 1u)) continue;
        out[(static_cast<size_t>(r) * n_pairs + cnt) * 2] = static_cast<int16_t>(i);
        out[(static_cast<size_t>(r) * n_pairs + cnt) * 2 + 1] = static_cast<int16_t>(j);
        ++cnt;
        taken[i >> 6] |= 1ull << (i & 63);
        taken[j >> 6] |= 1ull << (j & 63);
        used[q] = 1;
      }
    }
  }
  return PARO_OK;
}
