// paro_api.cu -- the C ABI declared in include/paro.h: argument checking, host-side
// transform preparation (paro_pack), kernel dispatch, NCCL all-gather.
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "../../include/paro.h"
#include "paro_internal.h"
#include "tile_layout.cuh"

namespace {

thread_local std::string g_err;

paro_status fail(paro_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

paro_status cuda_fail(cudaError_t e, const char* where) {
  return fail(PARO_ERR_CUDA, "%s: %s (%s)", where, cudaGetErrorName(e), cudaGetErrorString(e));
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

constexpr int kG = PARO_GROUP;

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

size_t dtype_bytes(paro_dtype d) { return d == PARO_F32 ? 4 : 2; }

size_t align256(size_t v) { return (v + 255) / 256 * 256; }

}  // namespace

namespace paro {
int set_error(int st, const char* msg) {
  g_err = msg;
  return st;
}
}  // namespace paro


// ---------------------------------------------------------------- bank-conflict-free rotation schedule
// One independent rotation = a perfect matching of the 128 channels of a group (absent
// slots are completed with identity pairs of the unpaired channels, cos = 1, sin = 0).
// The runtime kernels keep the group in shared memory and lane l of a warp updates the
// two pairs of slots (l, 0) and (l, 1): four gathers v[a0], v[b0], v[a1], v[b1] and four
// scatters per rotation.  With bank(ch) = ch % 32 each bank holds 4 channels, so the
// pairs form a 4-regular multigraph on the 32 banks.  Orienting it along an Euler
// circuit gives in = out = 2 at every bank; splitting the oriented edges into two
// perfect matchings (2-regular bipartite graph out-bank -> in-bank) yields, per slot,
// 32 pairs whose first channels hit 32 distinct banks and whose second channels do
// too -- every gather/scatter is conflict-free.  Swapping a pair's orientation is exact:
// (i, j, theta) == (j, i, -theta).  The slot order inside one independent rotation is
// irrelevant (Def. 2).
struct RotPair {
  int a, b;
  double c, s;
};

static void schedule_rotation(std::vector<RotPair> pairs, RotPair out[2][32]) {
  bool used[128] = {false};
  for (const RotPair& p : pairs) used[p.a] = used[p.b] = true;
  int pend = -1;
  for (int ch = 0; ch < 128; ++ch) {
    if (used[ch]) continue;
    if (pend < 0) {
      pend = ch;
    } else {
      pairs.push_back({pend, ch, 1.0, 0.0});
      pend = -1;
    }
  }
  const int E = static_cast<int>(pairs.size());  // 64
  std::vector<std::vector<std::pair<int, int>>> adj(32);  // (edge, other bank)
  for (int e = 0; e < E; ++e) {
    const int u = pairs[e].a & 31, v = pairs[e].b & 31;
    adj[u].push_back({e, v});
    adj[v].push_back({e, u});
  }
  std::vector<int> src(E, -1), dst(E, -1);  // oriented: bank src -> bank dst
  std::vector<bool> eused(E, false);
  std::vector<size_t> ptr(32, 0);
  for (int start = 0; start < 32; ++start) {
    // Hierholzer: walk unused edges, orienting each in traversal direction
    std::vector<int> stack{start};
    while (!stack.empty()) {
      const int x = stack.back();
      while (ptr[x] < adj[x].size() && eused[adj[x][ptr[x]].first]) ++ptr[x];
      if (ptr[x] == adj[x].size()) {
        stack.pop_back();
        continue;
      }
      const auto [e, y] = adj[x][ptr[x]];
      eused[e] = true;
      src[e] = x;
      dst[e] = y;
      stack.push_back(y);
    }
  }
  // split into two perfect matchings along the alternating cycles of out->in
  std::vector<std::vector<int>> outs(32), ins(32);
  for (int e = 0; e < E; ++e) {
    outs[src[e]].push_back(e);
    ins[dst[e]].push_back(e);
  }
  std::vector<int> slot(E, -1);
  for (int e0 = 0; e0 < E; ++e0) {
    if (slot[e0] >= 0) continue;
    int e = e0, s = 0;
    while (slot[e] < 0) {
      slot[e] = s;
      // partner at the same in-bank gets the other slot
      const std::vector<int>& in = ins[dst[e]];
      const int f = (in[0] == e) ? in[1] : in[0];
      if (slot[f] >= 0) break;
      slot[f] = 1 - s;
      // next: the other out-edge of f's source bank gets slot s again
      const std::vector<int>& ou = outs[src[f]];
      e = (ou[0] == f) ? ou[1] : ou[0];
    }
  }
  for (int e = 0; e < E; ++e) {
    const RotPair& p = pairs[e];
    RotPair r;
    // first element in bank src[e]
    if ((p.a & 31) == src[e] && ((p.b & 31) == dst[e])) {
      r = p;
    } else {
      r = {p.b, p.a, p.c, -p.s};
    }
    out[slot[e]][src[e]] = r;
  }
}

extern "C" {

const char* paro_last_error(void) { return g_err.c_str(); }
const char* paro_version(void) { return "paro-b200 0.1 (sm_100a)"; }

paro_status paro_pack_sizes(int64_t N, int64_t K, int32_t group, int32_t n_rot, paro_packed_sizes* out) {
  if (!out) return fail(PARO_ERR_INVALID_ARGUMENT, "paro_pack_sizes: out is NULL");
  if (N <= 0 || K <= 0) return fail(PARO_ERR_INVALID_ARGUMENT, "paro_pack_sizes: N and K must be > 0");
  if (group != kG) return fail(PARO_ERR_UNSUPPORTED, "paro_pack_sizes: group must be 128 (got %d)", group);
  if (K % kG) return fail(PARO_ERR_UNSUPPORTED, "paro_pack_sizes: K %% 128 != 0 (K=%lld)", (long long)K);
  if (n_rot < 0 || n_rot > PARO_MAX_ROT)
    return fail(PARO_ERR_UNSUPPORTED, "paro_pack_sizes: n_rot must be in [0, 8] (got %d)", n_rot);
  const int64_t G = K / kG;
  const int64_t tiles = ceil_div(N, int64_t(paro::TILE_ROWS)) * G;  // tile layout (tile_layout.cuh)
  out->codes = static_cast<size_t>(tiles * paro::TILE_CODE_BYTES);
  out->scales = static_cast<size_t>(tiles * paro::TILE_SCALE_BYTES);
  out->zeros = static_cast<size_t>(tiles * paro::TILE_ZERO_BYTES);
  out->rot_cs = static_cast<size_t>(G * n_rot * PARO_SLOTS * 8);
  out->rot_idx = static_cast<size_t>(G * n_rot * PARO_SLOTS * 2);
  out->svec = static_cast<size_t>(K * 4) + paro::KS_CTR_BYTES;  // s, then the K-split arrival counters
  return PARO_OK;
}

paro_status paro_pack(const void* W, const float* s, const float* theta, const int16_t* pairs, int64_t N, int64_t K,
                      int32_t group, int32_t n_rot, int32_t n_pairs, paro_packed* out, void* stream) {
  paro_packed_sizes sz;
  paro_status st = paro_pack_sizes(N, K, group, n_rot, &sz);
  if (st != PARO_OK) return st;
  if (!W || !s || !out) return fail(PARO_ERR_INVALID_ARGUMENT, "paro_pack: W, s, out must be non-NULL");
  if (n_rot > 0 && (!theta || !pairs))
    return fail(PARO_ERR_INVALID_ARGUMENT, "paro_pack: theta/pairs must be non-NULL when n_rot > 0");
  if (n_rot > 0 && (n_pairs < 1 || n_pairs > PARO_SLOTS))
    return fail(PARO_ERR_INVALID_ARGUMENT, "paro_pack: n_pairs must be in [1, 64] (got %d)", n_pairs);
  if (!out->codes || !out->scales || !out->zeros || !out->svec || (n_rot > 0 && (!out->rot_cs || !out->rot_idx)))
    return fail(PARO_ERR_INVALID_ARGUMENT, "paro_pack: packed buffers must be allocated");
  if (!aligned16(W) || !aligned16(out->codes) || !aligned16(out->scales) || !aligned16(out->zeros) ||
      !aligned16(out->svec) || !aligned16(out->rot_cs) || !aligned16(out->rot_idx))
    return fail(PARO_ERR_INVALID_ARGUMENT, "paro_pack: buffers must be 16-byte aligned");
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  const int64_t G = K / kG;
  const int L = n_rot, P = n_rot > 0 ? n_pairs : 0;

  // ---- copy the (small) transform to the host and validate it
  std::vector<float> hs(K), hth(static_cast<size_t>(G * L * P));
  std::vector<int16_t> hpr(static_cast<size_t>(G * L * P * 2));
  cudaError_t e = cudaMemcpyAsync(hs.data(), s, K * 4, cudaMemcpyDeviceToHost, cs);
  if (e == cudaSuccess && L > 0)
    e = cudaMemcpyAsync(hth.data(), theta, hth.size() * 4, cudaMemcpyDeviceToHost, cs);
  if (e == cudaSuccess && L > 0)
    e = cudaMemcpyAsync(hpr.data(), pairs, hpr.size() * 2, cudaMemcpyDeviceToHost, cs);
  if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
  if (e != cudaSuccess) return cuda_fail(e, "paro_pack: copying s/theta/pairs");
  for (int64_t k = 0; k < K; ++k)
    if (!std::isfinite(hs[k]) || !(hs[k] > 0.f))
      return fail(PARO_ERR_INVALID_ARGUMENT, "paro_pack: s[%lld] must be finite and > 0", (long long)k);
  // prepared transform: fp64 (cos, sin) for the fold, fp32 copies + u8 indices for the runtime
  // fold kernel tables are slot-major [G][L][64]; the runtime tables are records
  // [G][L][32 lanes][2 slots] (slot p = lane + 32 * s): 16-byte (cos0, sin0, cos1, sin1)
  // and 4-byte (i0, j0, i1, j1) per (group, rotation, lane), lane-contiguous.
  std::vector<double> cs64(static_cast<size_t>(G * L * PARO_SLOTS * 2), 0.0);
  std::vector<uint8_t> idx64(static_cast<size_t>(G * L * PARO_SLOTS * 2), 128);
  std::vector<float> cs32(static_cast<size_t>(G * L * PARO_SLOTS * 2), 0.f);
  std::vector<uint8_t> idx(static_cast<size_t>(G * L * PARO_SLOTS * 2), 128);
  auto lane_major = [&](int64_t g, int t, int p) -> size_t {
    return static_cast<size_t>(((g * L + t) * 32 + (p & 31)) * 2 + (p >> 5));
  };
  for (int64_t g = 0; g < G; ++g) {
    std::set<std::pair<int, int>> seen;
    for (int t = 0; t < L; ++t) {
      bool used[kG] = {false};
      std::vector<RotPair> layer;
      for (int p = 0; p < PARO_SLOTS; ++p) {
        const size_t o = static_cast<size_t>((g * L + t) * PARO_SLOTS + p);
        cs64[2 * o] = 1.0;
        if (p >= P) continue;
        const size_t src = static_cast<size_t>((g * L + t) * P + p);
        const int i = hpr[2 * src], j = hpr[2 * src + 1];
        if (i == -1 && j == -1) continue;  // absent slot (short rotation)
        if (i < 0 || j < 0 || i >= kG || j >= kG)
          return fail(PARO_ERR_PAIRS, "pairs[%lld,%d,%d] = (%d,%d) out of [0,128)", (long long)g, t, p, i, j);
        if (!(i < j)) return fail(PARO_ERR_PAIRS, "pairs[%lld,%d,%d] = (%d,%d): need i < j", (long long)g, t, p, i, j);
        if (used[i] || used[j])
          return fail(PARO_ERR_PAIRS, "rotation (%lld,%d) uses a channel twice (Definition 1)", (long long)g, t);
        used[i] = used[j] = true;
        if (!seen.insert({i, j}).second)
          return fail(PARO_ERR_PAIRS, "group %lld repeats pair (%d,%d) across rotations", (long long)g, i, j);
        const float th = hth[src];
        if (!std::isfinite(th))
          return fail(PARO_ERR_INVALID_ARGUMENT, "theta[%lld,%d,%d] is not finite", (long long)g, t, p);
        const double c = std::cos(static_cast<double>(th)), sn = std::sin(static_cast<double>(th));
        cs64[2 * o] = c;
        cs64[2 * o + 1] = sn;
        idx64[2 * o] = static_cast<uint8_t>(i);
        idx64[2 * o + 1] = static_cast<uint8_t>(j);
        layer.push_back({i, j, c, sn});
      }
      RotPair sched[2][32];
      schedule_rotation(layer, sched);
      for (int sl = 0; sl < 2; ++sl)
        for (int ln = 0; ln < 32; ++ln) {
          const size_t r = lane_major(g, t, ln + 32 * sl);
          const RotPair& q = sched[sl][ln];
          cs32[2 * r] = static_cast<float>(q.c);
          cs32[2 * r + 1] = static_cast<float>(q.s);
          idx[2 * r] = static_cast<uint8_t>(q.a);
          idx[2 * r + 1] = static_cast<uint8_t>(q.b);
        }
    }
  }
  // ---- device temporaries: fp64 (cos, sin) table, status word
  const size_t cs_bytes = cs64.size() * sizeof(double);
  const size_t tmp_bytes = align256(cs_bytes) + align256(idx64.size()) + 256;
  void* tmp = nullptr;
  e = cudaMallocAsync(&tmp, tmp_bytes, cs);
  if (e != cudaSuccess) return cuda_fail(e, "paro_pack: cudaMallocAsync");
  uint8_t* tb = static_cast<uint8_t*>(tmp);
  uint8_t* idx_dev = tb + align256(cs_bytes);
  int* status = reinterpret_cast<int*>(idx_dev + align256(idx64.size()));
  e = cudaMemsetAsync(status, 0, 4, cs);
  if (e == cudaSuccess && cs_bytes) e = cudaMemcpyAsync(tb, cs64.data(), cs_bytes, cudaMemcpyHostToDevice, cs);
  if (e == cudaSuccess && !idx64.empty())
    e = cudaMemcpyAsync(idx_dev, idx64.data(), idx64.size(), cudaMemcpyHostToDevice, cs);
  if (e == cudaSuccess && L > 0) e = cudaMemcpyAsync(out->rot_cs, cs32.data(), cs32.size() * 4, cudaMemcpyHostToDevice, cs);
  if (e == cudaSuccess && L > 0) e = cudaMemcpyAsync(out->rot_idx, idx.data(), idx.size(), cudaMemcpyHostToDevice, cs);
  if (e == cudaSuccess) e = cudaMemcpyAsync(out->svec, s, K * 4, cudaMemcpyDeviceToDevice, cs);
  if (e == cudaSuccess)  // the long-K decode split's arrival counters (every call leaves them zero)
    e = cudaMemsetAsync(static_cast<uint8_t*>(out->svec) + K * 4, 0, paro::KS_CTR_BYTES, cs);
  // zero the packed buffers: rows >= N of the last row block stay zero, zero points are
  // OR-ed in nibble by nibble
  if (e == cudaSuccess) e = cudaMemsetAsync(out->codes, 0, sz.codes, cs);
  if (e == cudaSuccess) e = cudaMemsetAsync(out->scales, 0, sz.scales, cs);
  if (e == cudaSuccess) e = cudaMemsetAsync(out->zeros, 0, sz.zeros, cs);
  if (e == cudaSuccess)
    e = paro::launch_pack(W, s, tb, idx_dev, N, K, L, out->codes, out->scales, out->zeros, status, cs);
  int hstatus = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&hstatus, status, 4, cudaMemcpyDeviceToHost, cs);
  cudaError_t e2 = cudaFreeAsync(tmp, cs);
  if (e == cudaSuccess) e = e2;
  if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
  if (e != cudaSuccess) return cuda_fail(e, "paro_pack");
  if (hstatus & 1) return fail(PARO_ERR_INVALID_ARGUMENT, "paro_pack: W (or the folded W) is not finite");
  if (hstatus & 2) return fail(PARO_ERR_INVALID_ARGUMENT, "paro_pack: a group's fp16 scale overflows");
  out->N = N;
  out->K = K;
  out->group = group;
  out->n_rot = n_rot;
  return PARO_OK;
}

static bool use_prefill(int64_t B, int64_t N, int64_t K, uint32_t flags) {
  if (flags & PARO_LINEAR_FORCE_GEMV) return false;
  if (!paro::prefill_supported(B, N, K)) return false;
  return (flags & PARO_LINEAR_FORCE_GEMM) || B > 16;
}

size_t paro_linear_workspace(int64_t B, int64_t N, int64_t K, int32_t n_rot, int32_t n_pairs, int32_t on_the_fly,
                             uint32_t flags) {
  (void)n_pairs;
  size_t ws = 0;
  if (on_the_fly && n_rot > 0) {
    const int64_t G = K / kG;
    ws += align256(static_cast<size_t>(G * n_rot * PARO_SLOTS * 8));
    ws += align256(static_cast<size_t>(G * n_rot * PARO_SLOTS * 2));
  }
  if (use_prefill(B, N, K, flags)) {
    ws += align256(static_cast<size_t>(B * K * 2));
    if (B >= paro::DENSE_XFORM_MIN_TOKENS) ws += align256(paro::transform_dense_ws_bytes(K));  // M rows
  }
  else if (B > 1 && paro::gemv1_enabled())  // decode, 2..16 tokens: pre-transformed x' (gemv1.cu)
    ws += paro::gemv1_xq_bytes(static_cast<int>(std::min<int64_t>(B, paro::GEMV1_MAX_B)), K);
  else if (B == 1 && paro::gemv1_enabled() && !(flags & 0x100u))  // one token, long K: cross-cluster K split
    ws += align256(paro::b1_ks_bytes(paro::b1_ks_slices(1, &N, K), N));
  return ws;
}


// transform tables to use for linear i of a decode launch (on-the-fly override or packed)
struct RotOverride {
  const float2* cs;
  const uchar2* idx;
  const float* s;
  int active;
};
static RotOverride rot_cs_override(const float2* cs, const uchar2* idx, const float* s, int on) {
  return RotOverride{cs, idx, s, on};
}

static paro_status decode_linears(const void* x, paro_dtype x_dtype, int64_t B, int n, const paro_packed* packed,
                                  RotOverride ov, const float* const* bias, void* const* y, paro_dtype y_dtype,
                                  int rotate, int pdl, int debug, int tcgen05, void* ws, size_t ws_bytes,
                                  cudaStream_t cs) {
  int64_t Ns[paro::GEMV_MAX_LIN];
  int Ls[paro::GEMV_MAX_LIN];
  for (int i = 0; i < n; ++i) {
    Ns[i] = packed[i].N;
    Ls[i] = packed[i].n_rot;
  }
  const int64_t K = packed[0].K;
  const size_t xe = 2, ye = dtype_bytes(y_dtype);
  paro::GemvConfig cfg;
  int planned_b = 0;
  // token count -> kernel (measured, tools/time_batch.py): the K-split kernel (gemv1.cu; B = 1:
  // gemv1_b1.cu) except B = 2 with K <= 3072 (the cluster-shared-transform kernel, gemv.cu)
#if PARO_DEBUG_KNOBS
  static const int small_b = [] {
    const char* e = getenv("PARO_G1_SMALLB");
    return e ? atoi(e) : 0;
  }();
#else
  constexpr int small_b = 0;
#endif
  // 2..4 tokens (tools/ab_smallb.sh, round 2, one-token transform tasks): the K-split kernel
  // wins or ties everywhere (N = 28672 x K = 4096 at B = 4: 15.5 vs 25.2 us) except B = 2 with a
  // short K (9728 x 2560: 8.2 vs 9.3 us), which keeps the cluster-shared-transform kernel
  const bool old_small = B == 2 && K <= 3072;
  bool k_split = !debug && paro::gemv1_enabled() && (B == 1 || B > 4 || !old_small || small_b || tcgen05);
  if (!k_split && !debug && paro::gemv1_enabled()) {  // the other kernel must be able to plan this shape
    const int bt0 = B <= 1 ? 1 : B <= 2 ? 2 : B <= 4 ? 4 : 8;
    const char* why0 = "";
    if (!paro::plan_gemv(bt0, n, Ns, Ls, K, rotate, &cfg, &why0)) k_split = true;
  }
  const int64_t tile_b = k_split ? paro::GEMV1_MAX_B : paro::GEMV_MAX_B;
  for (int64_t b0 = 0; b0 < B; b0 += tile_b) {
    const int live = static_cast<int>(std::min<int64_t>(tile_b, B - b0));
    if (k_split && live == 1) {  // one token: the one-launch kernel (gemv1_b1.cu)
      paro::B1Config c1;
      const char* why = "";
      // one linear, long K: the K range split over clusters when the workspace holds the row sums
      // (paro_linear_workspace reports them); the arrival counters live after s in packed svec
      float* ks_part = nullptr;
      uint32_t* ks_ctr = nullptr;
      if (B == 1 && n == 1) {
        const size_t kb = paro::b1_ks_bytes(paro::b1_ks_slices(1, Ns, K), Ns[0]);
        if (kb && ws && ws_bytes >= kb) {
          ks_part = static_cast<float*>(ws);
          ks_ctr = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(packed[0].svec) + K * 4);
        }
      }
      if (!paro::plan_gemv1_b1(1, n, Ns, K, rotate, ks_part, ks_ctr, &c1, &why))
        return fail(PARO_ERR_UNSUPPORTED, "paro_linear: %s", why);
      paro::B1Args& a = c1.a;
      a.x = static_cast<const uint8_t*>(x) + b0 * K * xe;
      a.x_bf16 = x_dtype == PARO_BF16;
      for (int i = 0; i < n; ++i) {
        paro::B1Linear& d = a.lin[i];
        d.codes = static_cast<const uint8_t*>(packed[i].codes);
        d.scales = static_cast<const uint8_t*>(packed[i].scales);
        d.zeros = static_cast<const uint8_t*>(packed[i].zeros);
        d.rot_cs = ov.active ? ov.cs : static_cast<const float2*>(packed[i].rot_cs);
        d.rot_idx = ov.active ? ov.idx : static_cast<const uchar2*>(packed[i].rot_idx);
        d.svec = ov.active ? ov.s : static_cast<const float*>(packed[i].svec);
        d.bias = bias ? bias[i] : nullptr;
        d.y = static_cast<uint8_t*>(y[i]) + b0 * packed[i].N * ye;
        d.L = packed[i].n_rot;
      }
      a.y_dtype = static_cast<int>(y_dtype);
      a.pdl = pdl;
      cudaError_t e = paro::launch_gemv1_b1(c1, cs);
      if (e != cudaSuccess) return cuda_fail(e, "paro_linear: decode GEMV (B=1) launch");
      continue;
    }
    if (k_split) {
      paro::Gemv1Config c1;
      const char* why = "";
      if (!paro::plan_gemv1(live, n, Ns, K, rotate, tcgen05, &c1, &why))
        return fail(PARO_ERR_UNSUPPORTED, "paro_linear: %s", why);
      paro::Gemv1Args& a = c1.a;
      paro::Gemv1Stage& S0 = a.st[0];
      S0.x = static_cast<const uint8_t*>(x) + b0 * K * xe;
      a.x_bf16 = x_dtype == PARO_BF16;
      for (int i = 0; i < n; ++i) {
        paro::Gemv1Linear& d = S0.lin[i];
        d.codes = static_cast<const uint8_t*>(packed[i].codes);
        d.scales = static_cast<const uint8_t*>(packed[i].scales);
        d.zeros = static_cast<const uint8_t*>(packed[i].zeros);
        d.rot_cs = ov.active ? ov.cs : static_cast<const float2*>(packed[i].rot_cs);
        d.rot_idx = ov.active ? ov.idx : static_cast<const uchar2*>(packed[i].rot_idx);
        d.svec = ov.active ? ov.s : static_cast<const float*>(packed[i].svec);
        d.bias = bias ? bias[i] : nullptr;
        d.y = static_cast<uint8_t*>(y[i]) + b0 * packed[i].N * ye;
        d.L = packed[i].n_rot;
      }
      a.y_dtype = static_cast<int>(y_dtype);
      a.pdl = pdl;
      if (live > 1) {  // x' of all tokens once, by a small transform kernel, into the workspace
        const size_t per = paro::gemv1_xq_bytes(live, K);
        if (!ws || ws_bytes < per * n)
          return fail(PARO_ERR_INVALID_ARGUMENT, "paro_linear: workspace too small (%zu < %zu)", ws_bytes, per * n);
        for (int i = 0; i < n; ++i) {
          uint8_t* base = static_cast<uint8_t*>(ws) + per * i;
          S0.lin[i].xq = base;
          S0.lin[i].xqs = reinterpret_cast<int2*>(base + static_cast<size_t>(K / kG) * paro::GEMV1_XQ_GROUP_BYTES);
        }
        cudaError_t e = paro::launch_gemv1_xform(c1, cs);
        if (e != cudaSuccess) return cuda_fail(e, "paro_linear: decode activation transform launch");
      }
      cudaError_t e = paro::launch_gemv1(c1, cs);
      if (e != cudaSuccess) return cuda_fail(e, "paro_linear: decode GEMV (B=1) launch");
      continue;
    }
    const int bt = live <= 1 ? 1 : live <= 2 ? 2 : live <= 4 ? 4 : 8;  // kernel token tile
    if (bt != planned_b) {
      const char* why = "";
      if (!paro::plan_gemv(bt, n, Ns, Ls, K, rotate, &cfg, &why)) return fail(PARO_ERR_UNSUPPORTED, "paro_linear: %s", why);
      planned_b = bt;
    }
    paro::GemvArgs& a = cfg.a;
    a.B = live;
    a.x = static_cast<const uint8_t*>(x) + b0 * K * xe;
    a.x_bf16 = x_dtype == PARO_BF16;
    for (int i = 0; i < n; ++i) {
      paro::GemvLinear& d = a.lin[i];
      d.codes = static_cast<const uint8_t*>(packed[i].codes);
      d.scales = static_cast<const uint8_t*>(packed[i].scales);
      d.zeros = static_cast<const uint8_t*>(packed[i].zeros);
      d.rot_cs = ov.active ? ov.cs : static_cast<const float2*>(packed[i].rot_cs);
      d.rot_idx = ov.active ? ov.idx : static_cast<const uchar2*>(packed[i].rot_idx);
      d.svec = ov.active ? ov.s : static_cast<const float*>(packed[i].svec);
      d.bias = bias ? bias[i] : nullptr;
      d.y = static_cast<uint8_t*>(y[i]) + b0 * packed[i].N * ye;
    }
    a.y_dtype = static_cast<int>(y_dtype);
    a.pdl = pdl;
    a.debug = debug;
    cudaError_t e = paro::launch_gemv(cfg, cs);
    if (e != cudaSuccess) return cuda_fail(e, "paro_linear: decode GEMV launch");
  }
  return PARO_OK;
}

static paro_status check_packed(const paro_packed* p) {
  if (!p) return fail(PARO_ERR_INVALID_ARGUMENT, "packed is NULL");
  if (p->group != kG) return fail(PARO_ERR_UNSUPPORTED, "packed->group must be 128");
  if (p->N <= 0 || p->K <= 0 || p->K % kG) return fail(PARO_ERR_SHAPE, "packed has invalid N/K");
  if (p->n_rot < 0 || p->n_rot > PARO_MAX_ROT) return fail(PARO_ERR_UNSUPPORTED, "packed->n_rot out of [0, 8]");
  if (!p->codes || !p->scales || !p->zeros || !p->svec || (p->n_rot > 0 && (!p->rot_cs || !p->rot_idx)))
    return fail(PARO_ERR_INVALID_ARGUMENT, "packed buffers must be non-NULL");
  if (!aligned16(p->codes) || !aligned16(p->scales) || !aligned16(p->zeros) || !aligned16(p->svec) ||
      !aligned16(p->rot_cs) || !aligned16(p->rot_idx))
    return fail(PARO_ERR_INVALID_ARGUMENT, "packed buffers must be 16-byte aligned");
  return PARO_OK;
}

paro_status paro_linear(const void* x, paro_dtype x_dtype, int64_t B, const paro_packed* packed, const float* s,
                        const float* theta, const int16_t* pairs, int32_t n_pairs, const float* bias, void* y,
                        paro_dtype y_dtype, uint32_t flags, void* workspace, size_t workspace_bytes, void* stream) {
  paro_status st = check_packed(packed);
  if (st != PARO_OK) return st;
  if (!x || !y) return fail(PARO_ERR_INVALID_ARGUMENT, "paro_linear: x and y must be non-NULL");
  if (B <= 0) return fail(PARO_ERR_INVALID_ARGUMENT, "paro_linear: B must be > 0");
  if (x_dtype != PARO_F16 && x_dtype != PARO_BF16)
    return fail(PARO_ERR_UNSUPPORTED, "paro_linear: x must be fp16 or bf16");
  if (y_dtype != PARO_F16 && y_dtype != PARO_BF16 && y_dtype != PARO_F32)
    return fail(PARO_ERR_UNSUPPORTED, "paro_linear: y must be fp16, bf16 or fp32");
  if (!aligned16(x) || !aligned16(y)) return fail(PARO_ERR_INVALID_ARGUMENT, "paro_linear: x, y must be 16-byte aligned");
  const int on_the_fly = (s || theta || pairs) ? 1 : 0;
  const int64_t N = packed->N, K = packed->K, G = K / kG;
  const int L = packed->n_rot;
  if (on_the_fly && (!s || (L > 0 && (!theta || !pairs))))
    return fail(PARO_ERR_INVALID_ARGUMENT, "paro_linear: give all of s/theta/pairs or none");
  if (on_the_fly && L > 0 && (n_pairs < 1 || n_pairs > PARO_SLOTS))
    return fail(PARO_ERR_INVALID_ARGUMENT, "paro_linear: n_pairs must be in [1, 64]");
  const size_t need = paro_linear_workspace(B, N, K, L, n_pairs, on_the_fly, flags);
  if (workspace_bytes < need || (need && !workspace))
    return fail(PARO_ERR_INVALID_ARGUMENT, "paro_linear: workspace too small (%zu < %zu)", workspace_bytes, need);
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  const int rotate = (flags & PARO_LINEAR_NO_ROTATION) ? 0 : 1;
  // on-the-fly tables are written by prepare_transform_kernel just before; the decode kernels
  // read them before their PDL wait, so the kernel after it is launched without PDL
  const int pdl = ((flags & PARO_LINEAR_PDL) && !on_the_fly) ? 1 : 0;
  const float2* rot_cs = static_cast<const float2*>(packed->rot_cs);
  const uchar2* rot_idx = static_cast<const uchar2*>(packed->rot_idx);
  const float* svec = static_cast<const float*>(packed->svec);
  uint8_t* wsp = static_cast<uint8_t*>(workspace);
  if (on_the_fly) {
    svec = s;
    if (L > 0) {
      float2* wcs = reinterpret_cast<float2*>(wsp);
      wsp += align256(static_cast<size_t>(G * L * PARO_SLOTS * 8));
      uchar2* widx = reinterpret_cast<uchar2*>(wsp);
      wsp += align256(static_cast<size_t>(G * L * PARO_SLOTS * 2));
      cudaError_t e = paro::launch_prepare_transform(theta, pairs, static_cast<int>(G), L, n_pairs, wcs, widx, cs);
      if (e != cudaSuccess) return cuda_fail(e, "paro_linear: prepare transform");
      rot_cs = wcs;
      rot_idx = widx;
    }
  }
  if (use_prefill(B, N, K, flags)) {
    void* xq = wsp;
    uint8_t* mws = wsp + align256(static_cast<size_t>(B * K * 2));
    // many tokens: the transform as a dense per-group contraction (misc.cu), else Givens passes
    cudaError_t e = (rotate && x_dtype == PARO_F16 && B >= paro::DENSE_XFORM_MIN_TOKENS)
                        ? paro::launch_transform_dense(x, x_dtype == PARO_BF16, B, K, L, svec, rot_cs, rot_idx, xq, mws,
                                                       pdl, 1, cs)
                        : paro::launch_transform(x, x_dtype == PARO_BF16, B, K, L, svec, rot_cs, rot_idx, rotate, xq,
                                                 pdl, 1, cs);
    if (e != cudaSuccess) return cuda_fail(e, "paro_linear: activation transform");
    e = paro::launch_prefill_gemm(xq, B, static_cast<const uint8_t*>(packed->codes),
                                  static_cast<const uint8_t*>(packed->scales), static_cast<const uint8_t*>(packed->zeros),
                                  bias, y, static_cast<int>(y_dtype), N, K, pdl, cs);
    if (e != cudaSuccess) return cuda_fail(e, "paro_linear: prefill GEMM");
    return PARO_OK;
  }
  // decode GEMV over token tiles
  const size_t used = static_cast<size_t>(wsp - static_cast<uint8_t*>(workspace));
  return decode_linears(x, x_dtype, B, 1, packed, rot_cs_override(rot_cs, rot_idx, svec, on_the_fly), &bias, &y,
                        y_dtype, rotate, pdl, (flags & 0x100u) ? 1 : 0, (flags & PARO_LINEAR_TCGEN05) ? 1 : 0, wsp,
                        workspace_bytes > used ? workspace_bytes - used : 0, cs);
}

paro_status paro_linear_multi(const void* x, paro_dtype x_dtype, int64_t B, int32_t n, const paro_packed* packed,
                              const float* const* bias, void* const* y, paro_dtype y_dtype, uint32_t flags,
                              void* workspace, size_t workspace_bytes, void* stream) {
  if (n < 1 || n > paro::GEMV_MAX_LIN || !packed || !y)
    return fail(PARO_ERR_INVALID_ARGUMENT, "paro_linear_multi: 1..4 linears, packed and y arrays required");
  for (int i = 0; i < n; ++i) {
    paro_status st = check_packed(&packed[i]);
    if (st != PARO_OK) return st;
    if (packed[i].K != packed[0].K) return fail(PARO_ERR_SHAPE, "paro_linear_multi: all linears must share K");
    if (!y[i] || !aligned16(y[i])) return fail(PARO_ERR_INVALID_ARGUMENT, "paro_linear_multi: y[%d] NULL/misaligned", i);
  }
  if (!x || !aligned16(x) || B <= 0) return fail(PARO_ERR_INVALID_ARGUMENT, "paro_linear_multi: bad x/B");
  if (x_dtype != PARO_F16 && x_dtype != PARO_BF16) return fail(PARO_ERR_UNSUPPORTED, "x must be fp16 or bf16");
  if (y_dtype != PARO_F16 && y_dtype != PARO_BF16 && y_dtype != PARO_F32)
    return fail(PARO_ERR_UNSUPPORTED, "y must be fp16, bf16 or fp32");
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  bool prefill = false;
  for (int i = 0; i < n; ++i) prefill = prefill || use_prefill(B, packed[i].N, packed[i].K, flags);
  if (prefill || n == 1) {  // prefill: one GEMM per linear (each with its own transform)
    for (int i = 0; i < n; ++i) {
      paro_status st = paro_linear(x, x_dtype, B, &packed[i], nullptr, nullptr, nullptr, 0, bias ? bias[i] : nullptr,
                                   y[i], y_dtype, flags, workspace, workspace_bytes, stream);
      if (st != PARO_OK) return st;
    }
    return PARO_OK;
  }
  const int rotate = (flags & PARO_LINEAR_NO_ROTATION) ? 0 : 1;
  const int pdl = (flags & PARO_LINEAR_PDL) ? 1 : 0;
  size_t need = 0;  // n x the per-linear decode workspace
  for (int i = 0; i < n; ++i)
    need = std::max(need, paro_linear_workspace(B, packed[i].N, packed[i].K, packed[i].n_rot, PARO_SLOTS, 0, flags));
  need *= static_cast<size_t>(n);
  if (workspace_bytes < need || (need && !workspace))
    return fail(PARO_ERR_INVALID_ARGUMENT, "paro_linear_multi: workspace too small (%zu < %zu)", workspace_bytes, need);
  return decode_linears(x, x_dtype, B, n, packed, rot_cs_override(nullptr, nullptr, nullptr, 0), bias, y, y_dtype,
                        rotate, pdl, (flags & 0x100u) ? 1 : 0, (flags & PARO_LINEAR_TCGEN05) ? 1 : 0, workspace,
                        workspace_bytes, cs);
}

// ---------------------------------------------------------------- persistent decode chain
// workspace header: grid-barrier epoch word + one arrival flag per CTA (zero before first use)
constexpr size_t kChainHdr = 8192;
static size_t chain_xq_bytes(int64_t B, int32_t n_stages, const paro_chain_stage* stages) {
  if (B <= 1) return 0;
  int64_t Kmax = 0;
  for (int s = 0; s < n_stages; ++s)
    for (int i = 0; i < stages[s].n; ++i) Kmax = std::max<int64_t>(Kmax, stages[s].packed[i].K);
  return paro::gemv1_xq_bytes(static_cast<int>(std::min<int64_t>(B, paro::GEMV1_MAX_B)), Kmax);
}

size_t paro_linear_chain_workspace(int64_t B, int32_t n_stages, const paro_chain_stage* stages) {
  if (n_stages < 1 || !stages) return 0;
  for (int s = 0; s < n_stages; ++s)
    if (stages[s].n < 1 || stages[s].n > paro::GEMV_MAX_LIN || !stages[s].packed) return 0;
  // grid-barrier words + (B > 1) one x'-digit buffer per linear slot, shared by the stages
  return kChainHdr + align256(chain_xq_bytes(B, n_stages, stages) * paro::GEMV_MAX_LIN);
}

paro_status paro_linear_chain(int32_t n_stages, const paro_chain_stage* stages, paro_dtype x_dtype, int64_t B,
                              paro_dtype y_dtype, uint32_t flags, void* workspace, size_t workspace_bytes,
                              void* stream) {
  if (n_stages < 1 || !stages) return fail(PARO_ERR_INVALID_ARGUMENT, "paro_linear_chain: n_stages >= 1 and stages required");
  if (B < 1 || B > paro::GEMV1_MAX_B) return fail(PARO_ERR_UNSUPPORTED, "paro_linear_chain: decode chains take 1..16 tokens");
  if (x_dtype != PARO_F16 && x_dtype != PARO_BF16) return fail(PARO_ERR_UNSUPPORTED, "x must be fp16 or bf16");
  if (y_dtype != PARO_F16 && y_dtype != PARO_BF16 && y_dtype != PARO_F32)
    return fail(PARO_ERR_UNSUPPORTED, "y must be fp16, bf16 or fp32");
  for (int s = 0; s < n_stages; ++s) {
    const paro_chain_stage& S = stages[s];
    if (S.n < 1 || S.n > paro::GEMV_MAX_LIN || !S.packed || !S.y)
      return fail(PARO_ERR_INVALID_ARGUMENT, "paro_linear_chain: stage %d needs 1..4 linears, packed and y", s);
    if (!S.x || !aligned16(S.x)) return fail(PARO_ERR_INVALID_ARGUMENT, "paro_linear_chain: stage %d x NULL/misaligned", s);
    for (int i = 0; i < S.n; ++i) {
      paro_status st = check_packed(&S.packed[i]);
      if (st != PARO_OK) return st;
      if (S.packed[i].K != S.packed[0].K) return fail(PARO_ERR_SHAPE, "paro_linear_chain: stage %d linears must share K", s);
      if (!S.y[i] || !aligned16(S.y[i]))
        return fail(PARO_ERR_INVALID_ARGUMENT, "paro_linear_chain: stage %d y[%d] NULL/misaligned", s, i);
    }
  }
  const size_t need = paro_linear_chain_workspace(B, n_stages, stages);
  if (!workspace || workspace_bytes < need || !aligned16(workspace))
    return fail(PARO_ERR_INVALID_ARGUMENT, "paro_linear_chain: workspace too small (%zu < %zu) or misaligned",
                workspace_bytes, need);
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  const int rotate = (flags & PARO_LINEAR_NO_ROTATION) ? 0 : 1;
  const size_t xe = dtype_bytes(x_dtype), ye = dtype_bytes(y_dtype);
  const size_t xq_per = chain_xq_bytes(B, n_stages, stages);
  uint8_t* wsb = static_cast<uint8_t*>(workspace);
  // chains longer than one argument block run as several launches (the first with the caller's
  // PDL choice, the later ones always PDL-chained: they only wait for the previous launch)
  for (int s0 = 0; s0 < n_stages; s0 += paro::CHAIN_MAX_STAGES) {
    const int ns = std::min(paro::CHAIN_MAX_STAGES, n_stages - s0);
    int nl[paro::CHAIN_MAX_STAGES];
    int64_t Ns[paro::CHAIN_MAX_STAGES][paro::GEMV_MAX_LIN] = {};
    int64_t Ks[paro::CHAIN_MAX_STAGES];
    for (int s = 0; s < ns; ++s) {
      const paro_chain_stage& S = stages[s0 + s];
      nl[s] = S.n;
      Ks[s] = S.packed[0].K;
      for (int i = 0; i < S.n; ++i) Ns[s][i] = S.packed[i].N;
    }
    paro::Gemv1Config c;
    const char* why = "";
    if (!paro::plan_gemv1_chain(static_cast<int>(B), ns, nl, Ns, Ks, rotate, (flags & PARO_LINEAR_TCGEN05) ? 1 : 0, &c,
                                &why))
      return fail(PARO_ERR_UNSUPPORTED, "paro_linear_chain: %s", why);
    paro::Gemv1Args& a = c.a;
    a.x_bf16 = x_dtype == PARO_BF16;
    a.y_dtype = static_cast<int>(y_dtype);
    a.pdl = (s0 > 0 || (flags & PARO_LINEAR_PDL)) ? 1 : 0;
    a.gbar = reinterpret_cast<uint32_t*>(wsb);
    for (int s = 0; s < ns; ++s) {
      const paro_chain_stage& S = stages[s0 + s];
      paro::Gemv1Stage& T = a.st[s];
      T.x = S.x;
      for (int i = 0; i < S.n; ++i) {
        const paro_packed& p = S.packed[i];
        paro::Gemv1Linear& d = T.lin[i];
        d.codes = static_cast<const uint8_t*>(p.codes);
        d.scales = static_cast<const uint8_t*>(p.scales);
        d.zeros = static_cast<const uint8_t*>(p.zeros);
        d.rot_cs = static_cast<const float2*>(p.rot_cs);
        d.rot_idx = static_cast<const uchar2*>(p.rot_idx);
        d.svec = static_cast<const float*>(p.svec);
        d.bias = S.bias ? S.bias[i] : nullptr;
        d.y = S.y[i];
        d.L = p.n_rot;
        if (B > 1) {
          uint8_t* base = wsb + kChainHdr + xq_per * i;
          d.xq = base;
          d.xqs = reinterpret_cast<int2*>(base + static_cast<size_t>(p.K / kG) * paro::GEMV1_XQ_GROUP_BYTES);
        }
      }
    }
    (void)xe;
    (void)ye;
    if (B > 1) {
      cudaError_t e = paro::launch_gemv1_xform(c, cs);
      if (e != cudaSuccess) return cuda_fail(e, "paro_linear_chain: stage-0 activation transform launch");
    }
    cudaError_t e = paro::launch_gemv1(c, cs);
    if (e != cudaSuccess) return cuda_fail(e, "paro_linear_chain: decode chain launch");
  }
  return PARO_OK;
}

paro_status paro_transform_activations(const void* x, paro_dtype x_dtype, int64_t B, const paro_packed* packed,
                                       void* x_out, void* stream) {
  paro_status st = check_packed(packed);
  if (st != PARO_OK) return st;
  if (!x || !x_out || B <= 0) return fail(PARO_ERR_INVALID_ARGUMENT, "paro_transform_activations: bad x/x_out/B");
  if (x_dtype != PARO_F16 && x_dtype != PARO_BF16) return fail(PARO_ERR_UNSUPPORTED, "x must be fp16 or bf16");
  cudaError_t e = paro::launch_transform(x, x_dtype == PARO_BF16, B, packed->K, packed->n_rot,
                                         static_cast<const float*>(packed->svec),
                                         static_cast<const float2*>(packed->rot_cs),
                                         static_cast<const uchar2*>(packed->rot_idx), 1, x_out, 0, 0,
                                         static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "paro_transform_activations");
  return PARO_OK;
}

size_t paro_transform_dense_workspace(int64_t K) { return paro::transform_dense_ws_bytes(K); }

paro_status paro_transform_activations_dense(const void* x, paro_dtype x_dtype, int64_t B, const paro_packed* packed,
                                             void* x_out, void* workspace, size_t workspace_bytes, void* stream) {
  paro_status st = check_packed(packed);
  if (st != PARO_OK) return st;
  if (!x || !x_out || B <= 0) return fail(PARO_ERR_INVALID_ARGUMENT, "paro_transform_activations_dense: bad x/x_out/B");
  if (x_dtype != PARO_F16) return fail(PARO_ERR_UNSUPPORTED, "paro_transform_activations_dense: x must be fp16");
  if (!aligned16(x) || !aligned16(x_out) || !aligned16(workspace))
    return fail(PARO_ERR_INVALID_ARGUMENT, "paro_transform_activations_dense: x, x_out, workspace must be 16-byte aligned");
  if (!workspace || workspace_bytes < paro::transform_dense_ws_bytes(packed->K))
    return fail(PARO_ERR_INVALID_ARGUMENT, "paro_transform_activations_dense: workspace too small (%zu < %zu)",
                workspace_bytes, paro::transform_dense_ws_bytes(packed->K));
  cudaError_t e = paro::launch_transform_dense(x, x_dtype == PARO_BF16, B, packed->K, packed->n_rot,
                                               static_cast<const float*>(packed->svec),
                                               static_cast<const float2*>(packed->rot_cs),
                                               static_cast<const uchar2*>(packed->rot_idx), x_out, workspace, 0, 0,
                                               static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "paro_transform_activations_dense");
  return PARO_OK;
}

paro_status paro_copy(void* dst, const void* src, size_t bytes, uint32_t flags, void* stream) {
  if (!dst || !src) return fail(PARO_ERR_INVALID_ARGUMENT, "paro_copy: NULL dst/src");
  if (bytes % 16 || !aligned16(dst) || !aligned16(src))
    return fail(PARO_ERR_INVALID_ARGUMENT, "paro_copy: bytes and both pointers must be multiples of 16");
  if (!bytes) return PARO_OK;
  cudaError_t e = paro::launch_copy16(dst, src, bytes, (flags & PARO_LINEAR_PDL) ? 1 : 0, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "paro_copy");
  return PARO_OK;
}

paro_status paro_fwht(const void* x, paro_dtype x_dtype, int64_t T, int64_t n, const float* signs, float scale,
                      void* y, void* stream) {
  if (!x || !y || T <= 0) return fail(PARO_ERR_INVALID_ARGUMENT, "paro_fwht: bad x/y/T");
  if (!aligned16(x) || !aligned16(y) || (signs && !aligned16(signs)))
    return fail(PARO_ERR_INVALID_ARGUMENT, "paro_fwht: x, y, signs must be 16-byte aligned");
  if (x_dtype != PARO_F16 && x_dtype != PARO_BF16) return fail(PARO_ERR_UNSUPPORTED, "paro_fwht: x must be fp16 or bf16");
  if (n < 256 || n > 16384 || (n & (n - 1)))
    return fail(PARO_ERR_UNSUPPORTED, "paro_fwht: n must be a power of two in [256, 16384]");
  cudaError_t e = paro::launch_fwht(x, x_dtype == PARO_BF16, T, n, signs, scale, y, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "paro_fwht");
  return PARO_OK;
}

paro_status paro_unpack_logical(const paro_packed* packed, void* codes_u8, void* scales_f16, void* zeros_u8,
                                void* stream) {
  paro_status st = check_packed(packed);
  if (st != PARO_OK) return st;
  if (!codes_u8 || !scales_f16 || !zeros_u8) return fail(PARO_ERR_INVALID_ARGUMENT, "paro_unpack_logical: NULL output");
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  const int64_t N = packed->N, K = packed->K, G = K / kG;
  (void)G;
  cudaError_t e = paro::launch_unpack(static_cast<const uint8_t*>(packed->codes),
                                      static_cast<const uint8_t*>(packed->scales),
                                      static_cast<const uint8_t*>(packed->zeros), N, K, static_cast<uint8_t*>(codes_u8),
                                      static_cast<uint8_t*>(scales_f16), static_cast<uint8_t*>(zeros_u8), cs);
  if (e != cudaSuccess) return cuda_fail(e, "paro_unpack_logical");
  return PARO_OK;
}

// ============================================================================ NCCL (dlopen)
typedef struct {
  char internal[PARO_NCCL_UNIQUE_ID_BYTES];
} nccl_uid_t;
typedef int (*nccl_get_uid_fn)(nccl_uid_t*);
typedef int (*nccl_init_rank_fn)(void**, int, nccl_uid_t, int);
typedef int (*nccl_destroy_fn)(void*);
typedef int (*nccl_allgather_fn)(const void*, void*, size_t, int, void*, cudaStream_t);
typedef const char* (*nccl_errstr_fn)(int);
typedef int (*nccl_async_err_fn)(void*, int*);

static struct {
  std::once_flag once;
  void* h = nullptr;
  nccl_get_uid_fn get_uid = nullptr;
  nccl_init_rank_fn init_rank = nullptr;
  nccl_destroy_fn destroy = nullptr;
  nccl_allgather_fn allgather = nullptr;
  nccl_errstr_fn errstr = nullptr;
  nccl_async_err_fn async_err = nullptr;
} g_nccl;

static bool nccl_load() {
  std::call_once(g_nccl.once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      g_nccl.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
      if (!g_nccl.h) g_nccl.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (g_nccl.h) break;
    }
    if (!g_nccl.h) return;
    g_nccl.get_uid = reinterpret_cast<nccl_get_uid_fn>(dlsym(g_nccl.h, "ncclGetUniqueId"));
    g_nccl.init_rank = reinterpret_cast<nccl_init_rank_fn>(dlsym(g_nccl.h, "ncclCommInitRank"));
    g_nccl.destroy = reinterpret_cast<nccl_destroy_fn>(dlsym(g_nccl.h, "ncclCommDestroy"));
    g_nccl.allgather = reinterpret_cast<nccl_allgather_fn>(dlsym(g_nccl.h, "ncclAllGather"));
    g_nccl.errstr = reinterpret_cast<nccl_errstr_fn>(dlsym(g_nccl.h, "ncclGetErrorString"));
    g_nccl.async_err = reinterpret_cast<nccl_async_err_fn>(dlsym(g_nccl.h, "ncclCommGetAsyncError"));
  });
  return g_nccl.get_uid && g_nccl.init_rank && g_nccl.destroy && g_nccl.allgather && g_nccl.async_err;
}

// Errors NCCL detects asynchronously (a peer died, a network / NVLink failure) are only
// reported through ncclCommGetAsyncError; surface them as PARO_ERR_NCCL on the next call.
static int nccl_async_error(void* comm) {
  int ar = 0;
  const int r = g_nccl.async_err(comm, &ar);
  return r ? r : ar;
}

static paro_status nccl_fail(int r, const char* where) {
  return fail(PARO_ERR_NCCL, "%s: nccl error %d (%s)", where, r, g_nccl.errstr ? g_nccl.errstr(r) : "?");
}

paro_status paro_comm_unique_id(void* uid) {
  if (!uid) return fail(PARO_ERR_INVALID_ARGUMENT, "paro_comm_unique_id: NULL");
  if (!nccl_load()) return fail(PARO_ERR_NCCL, "libnccl.so.2 could not be loaded");
  nccl_uid_t u;
  int r = g_nccl.get_uid(&u);
  if (r) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(uid, &u, sizeof(u));
  return PARO_OK;
}

paro_status paro_comm_init(const void* uid, int32_t rank, int32_t world, void** comm) {
  if (!uid || !comm || world < 1 || rank < 0 || rank >= world)
    return fail(PARO_ERR_INVALID_ARGUMENT, "paro_comm_init: bad arguments");
  if (!nccl_load()) return fail(PARO_ERR_NCCL, "libnccl.so.2 could not be loaded");
  nccl_uid_t u;
  std::memcpy(&u, uid, sizeof(u));
  int r = g_nccl.init_rank(comm, world, u, rank);
  if (r) return nccl_fail(r, "ncclCommInitRank");
  return PARO_OK;
}

paro_status paro_comm_check(void* comm) {
  if (!comm) return fail(PARO_ERR_INVALID_ARGUMENT, "paro_comm_check: NULL comm");
  if (!nccl_load()) return fail(PARO_ERR_NCCL, "libnccl.so.2 could not be loaded");
  if (int ar = nccl_async_error(comm)) return nccl_fail(ar, "ncclCommGetAsyncError");
  return PARO_OK;
}

paro_status paro_comm_destroy(void* comm) {
  if (!comm) return PARO_OK;
  if (!nccl_load()) return fail(PARO_ERR_NCCL, "libnccl.so.2 could not be loaded");
  int r = g_nccl.destroy(comm);
  if (r) return nccl_fail(r, "ncclCommDestroy");
  return PARO_OK;
}

size_t paro_linear_allgather_workspace(int64_t B, int64_t N_shard, int64_t K, int32_t world, paro_dtype y_dtype,
                                       uint32_t flags) {
  size_t ws = align256(static_cast<size_t>(B * N_shard) * dtype_bytes(y_dtype));  // local y
  if (B > 1) ws += align256(static_cast<size_t>(world) * B * N_shard * dtype_bytes(y_dtype));  // rank-major gather
  ws += paro_linear_workspace(B, N_shard, K, PARO_MAX_ROT, PARO_SLOTS, 0, flags);
  return ws;
}

paro_status paro_linear_allgather(const void* x, paro_dtype x_dtype, int64_t B, const paro_packed* packed_shard,
                                  const float* bias_shard, void* y_full, paro_dtype y_dtype, uint32_t flags,
                                  void* workspace, size_t workspace_bytes, void* comm, int32_t rank, int32_t world,
                                  void* stream) {
  paro_status st = check_packed(packed_shard);
  if (st != PARO_OK) return st;
  if (!comm || world < 1 || rank < 0 || rank >= world)
    return fail(PARO_ERR_INVALID_ARGUMENT, "paro_linear_allgather: bad comm/rank/world");
  if (!y_full || !workspace) return fail(PARO_ERR_INVALID_ARGUMENT, "paro_linear_allgather: NULL y_full/workspace");
  const int64_t Ns = packed_shard->N, K = packed_shard->K;
  const size_t need = paro_linear_allgather_workspace(B, Ns, K, world, y_dtype, flags);
  if (workspace_bytes < need)
    return fail(PARO_ERR_INVALID_ARGUMENT, "paro_linear_allgather: workspace too small (%zu < %zu)", workspace_bytes,
                need);
  if (!nccl_load()) return fail(PARO_ERR_NCCL, "libnccl.so.2 could not be loaded");
  if (int ar = nccl_async_error(comm)) return nccl_fail(ar, "ncclCommGetAsyncError (before the all-gather)");
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  const size_t ye = dtype_bytes(y_dtype);
  uint8_t* wsp = static_cast<uint8_t*>(workspace);
  uint8_t* y_local = wsp;
  wsp += align256(static_cast<size_t>(B * Ns) * ye);
  uint8_t* gather = nullptr;
  if (B > 1) {
    gather = wsp;
    wsp += align256(static_cast<size_t>(world) * B * Ns * ye);
  }
  const size_t rest = workspace_bytes - static_cast<size_t>(wsp - static_cast<uint8_t*>(workspace));
  st = paro_linear(x, x_dtype, B, packed_shard, nullptr, nullptr, nullptr, 0, bias_shard, y_local, y_dtype, flags, wsp,
                   rest, stream);
  if (st != PARO_OK) return st;
  // all-gather y over NVLink/NVSwitch on the same stream (rank-major [world][B][Ns])
  int r = g_nccl.allgather(y_local, B > 1 ? gather : y_full, static_cast<size_t>(B * Ns) * ye, /*ncclInt8*/ 0, comm,
                           cs);
  if (r) return nccl_fail(r, "ncclAllGather");
  if (int ar = nccl_async_error(comm)) return nccl_fail(ar, "ncclCommGetAsyncError");
  if (B > 1) {
    cudaError_t e = paro::launch_permute_gather(gather, y_full, world, B, Ns, static_cast<int>(ye), cs);
    if (e != cudaSuccess) return cuda_fail(e, "paro_linear_allgather: permute");
  }
  return PARO_OK;
}

// ---------------------------------------------------------------- NVLink-native all-gather (P2P)
static size_t p2p_y_bytes(int64_t B, int64_t N_full, paro_dtype y_dtype) {
  return align256(static_cast<size_t>(B * N_full) * dtype_bytes(y_dtype));
}

size_t paro_p2p_buffer_bytes(int64_t B, int64_t N_full, paro_dtype y_dtype, int32_t world) {
  if (B < 1 || N_full < 1 || world < 1 || world > paro::PARO_P2P_MAX_WORLD) return 0;
  return p2p_y_bytes(B, N_full, y_dtype) + 256;  // + flags[world], epoch, CTA counter
}

paro_status paro_ipc_get_handle(const void* dev_ptr, void* handle) {
  if (!dev_ptr || !handle) return fail(PARO_ERR_INVALID_ARGUMENT, "paro_ipc_get_handle: NULL argument");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr));
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
  std::memcpy(handle, &h, sizeof(h));
  return PARO_OK;
}

paro_status paro_ipc_open_handle(const void* handle, void** dev_ptr) {
  if (!dev_ptr || !handle) return fail(PARO_ERR_INVALID_ARGUMENT, "paro_ipc_open_handle: NULL argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
  return PARO_OK;
}

paro_status paro_ipc_close_handle(void* dev_ptr) {
  cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcCloseMemHandle");
  return PARO_OK;
}

paro_status paro_linear_allgather_p2p(const void* x, paro_dtype x_dtype, int64_t B, const paro_packed* packed_shard,
                                      const float* bias_shard, paro_dtype y_dtype, uint32_t flags,
                                      void* const* peer_bufs, int32_t rank, int32_t world, void* stream) {
  paro_status st = check_packed(packed_shard);
  if (st != PARO_OK) return st;
  if (B != 1) return fail(PARO_ERR_UNSUPPORTED, "paro_linear_allgather_p2p: one token per call (decode)");
  if (world < 1 || world > paro::PARO_P2P_MAX_WORLD || rank < 0 || rank >= world || !peer_bufs)
    return fail(PARO_ERR_INVALID_ARGUMENT, "paro_linear_allgather_p2p: bad rank/world/peer_bufs");
  for (int p = 0; p < world; ++p)
    if (!peer_bufs[p] || !aligned16(peer_bufs[p]))
      return fail(PARO_ERR_INVALID_ARGUMENT, "paro_linear_allgather_p2p: peer buffer %d NULL/misaligned", p);
  if (!x || !aligned16(x)) return fail(PARO_ERR_INVALID_ARGUMENT, "paro_linear_allgather_p2p: bad x");
  if (x_dtype != PARO_F16 && x_dtype != PARO_BF16) return fail(PARO_ERR_UNSUPPORTED, "x must be fp16 or bf16");
  if (y_dtype != PARO_F16 && y_dtype != PARO_BF16 && y_dtype != PARO_F32)
    return fail(PARO_ERR_UNSUPPORTED, "y must be fp16, bf16 or fp32");
  const int64_t Ns = packed_shard->N, K = packed_shard->K, N_full = Ns * world;
  paro::B1Config c;
  const char* why = "";
  if (!paro::plan_gemv1_b1(1, 1, &Ns, K, (flags & PARO_LINEAR_NO_ROTATION) ? 0 : 1, nullptr, nullptr, &c, &why))
    return fail(PARO_ERR_UNSUPPORTED, "paro_linear_allgather_p2p: %s", why);
  paro::B1Args& a = c.a;
  a.x = x;
  a.x_bf16 = x_dtype == PARO_BF16;
  paro::B1Linear& d = a.lin[0];
  d.codes = static_cast<const uint8_t*>(packed_shard->codes);
  d.scales = static_cast<const uint8_t*>(packed_shard->scales);
  d.zeros = static_cast<const uint8_t*>(packed_shard->zeros);
  d.rot_cs = static_cast<const float2*>(packed_shard->rot_cs);
  d.rot_idx = static_cast<const uchar2*>(packed_shard->rot_idx);
  d.svec = static_cast<const float*>(packed_shard->svec);
  d.bias = bias_shard;
  d.y = peer_bufs[rank];
  d.L = packed_shard->n_rot;
  a.y_dtype = static_cast<int>(y_dtype);
  a.pdl = (flags & PARO_LINEAR_PDL) ? 1 : 0;
  const size_t yb = p2p_y_bytes(1, N_full, y_dtype);
  a.p2p = 1;
  a.world = world;
  a.rank = rank;
  a.y_ld = N_full;
  a.y_col0 = static_cast<int64_t>(rank) * Ns;
  for (int p = 0; p < world; ++p) {
    a.peer_y[p] = peer_bufs[p];
    a.peer_flags[p] = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(peer_bufs[p]) + yb);
  }
  uint32_t* local_flags = a.peer_flags[rank];
  uint32_t* epoch = local_flags + 32;
  a.epoch = epoch;
  a.done_ctr = local_flags + 48;
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  cudaError_t e = paro::launch_gemv1_b1(c, cs);
  if (e == cudaSuccess) e = paro::launch_p2p_wait(local_flags, epoch, world, 0, cs);
  if (e != cudaSuccess) return cuda_fail(e, "paro_linear_allgather_p2p");
  return PARO_OK;
}

}  // extern "C"
