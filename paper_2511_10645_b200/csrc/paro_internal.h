// paro_internal.h -- declarations shared by the host API and the kernels (not installed).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace paro {

// thread-local error message of paro_last_error(); returns st
int set_error(int st, const char* msg);

// ---------------------------------------------------------------- pack
cudaError_t launch_pack(const void* W, const float* s, const void* cs64, const void* idx, int64_t N, int64_t K, int L,
                        void* codes, void* scales, void* zeros, int* status, cudaStream_t st);

// ---------------------------------------------------------------- decode GEMV
constexpr int GEMV_MAX_LIN = 4;  // linears sharing one activation in a single launch
constexpr int GEMV_MAX_B = 8;    // tokens per decode launch (the MMA's N = 8 columns)

// One linear of a (multi-)linear decode launch: its CTAs are [cta_begin, cta_begin + n_ctas)
// (whole clusters); cluster c owns rb_base + (c < rb_extra) consecutive 16-row blocks.
struct GemvLinear {
  const uint8_t* codes;   // tiles (tile_layout.cuh)
  const uint8_t* scales;
  const uint8_t* zeros;
  const float2* rot_cs;
  const uchar2* rot_idx;
  const float* svec;
  const float* bias;
  void* y;  // [B][N]
  int N, L;
  int cta_begin, n_ctas, rb_base, rb_extra;
};

struct GemvArgs {
  const void* x;  // [B][K] fp16 / bf16 (shared by all linears of the launch)
  int x_bf16;
  int B;          // tokens in this launch (1..8)
  int n_lin;
  GemvLinear lin[GEMV_MAX_LIN];
  int y_dtype;
  int K, G;
  int rotate;
  int pdl;
  int debug;        // record a per-CTA event timeline (g_paro_timeline)
  int xfirst;       // producer waits until the transform warps have issued their loads
  int early_stages; // under PDL: weight stages requested before that
  int stagger;      // experiment: stages issued (and the first awaited) before the rest of the ring
  int NW;           // compute warps
  int TPS;          // tiles per ring stage
  int scr_groups;   // transform groups per warp in lockstep (1 or 2)
  int S;            // ring depth
  int R_max;        // row blocks a CTA's tile range can touch
  uint32_t slot_bytes, sc_off, z_off;  // per-stage slot layout
  uint32_t off_u, off_xs, off_scr, off_part, off_recv, off_ring, off_bar, smem_total;
};

struct GemvConfig {
  int BT, NW, CL, grid;  // BT: compile-time token tile of the kernel instance
  bool IM;               // integer tensor-core (IMMA) instance (BT <= 2)
  GemvArgs a;
};

// Plan a launch (pure host arithmetic plus cached device / occupancy queries).
// n_lin linears of widths Ns[i] and rotation counts Ls[i] sharing K (and x); B = token tile
// (1, 2, 4 or 8); the launch sets cfg.a.B <= B live tokens.
bool plan_gemv(int B, int n_lin, const int64_t* Ns, const int* Ls, int64_t K, int rotate, GemvConfig* cfg,
               const char** why);
cudaError_t launch_gemv(const GemvConfig& cfg, cudaStream_t st);

// ---------------------------------------------------------------- decode GEMV, K-split (gemv1.cu)
// A launch runs a CHAIN of stages (one stage = one multi-linear GEMV whose linears share x);
// stage s + 1 starts after every CTA finished stage s (grid-wide barrier), so its x may be an
// earlier stage's y.  A single paro_linear / paro_linear_multi call is a one-stage chain.
// In stage s, cluster c of linear i owns rb_base + (c < rb_extra) consecutive 32-row blocks;
// CTA k of a cluster of CL owns the groups [k G / CL, (k + 1) G / CL) of those rows (K-split).
struct Gemv1Linear {
  const uint8_t* codes;
  const uint8_t* scales;
  const uint8_t* zeros;
  const float2* rot_cs;
  const uchar2* rot_idx;
  const float* svec;
  const float* bias;
  void* y;  // [B][N]
  uint8_t* xq;  // B > 1: pre-transformed x' digits [G][NB][4][8][4][8 B] (workspace)
  int2* xqs;    // B > 1: per (group, token) (sum x'fix, 2^(E-14)) [G][BT]
  int N, L;
  int cta_begin, rb_base, rb_extra;
};

constexpr int GEMV1_MAX_B = 16;       // tokens per launch of the K-split kernel
constexpr int CHAIN_MAX_STAGES = 16;  // stages per persistent launch (longer chains: several launches)

struct Gemv1Stage {
  const void* x;  // [B][K] fp16 / bf16
  int n_lin, K, G;
  int n_cta;      // CTAs with work in this stage (whole clusters); the others only pass the barriers
  int R_max;      // rows of the largest cluster (per-warp partial stride)
  int RRmax;      // rows per owner CTA (reduction)
  int atom;       // B = 1: row partials by shared atomics (clusters with too many rows)
  int xq_in_kernel;  // B > 1: x' digits computed inside the launch (x is an earlier stage's y)
  Gemv1Linear lin[GEMV_MAX_LIN];
};

template <int MS>
struct Gemv1ArgsT {
  int x_bf16;
  int B;  // tokens (1..16)
  int umma;  // B > 1: tiles on the tcgen05 tensor cores (kind::i8, TMEM) instead of mma.sync
  int y_dtype;
  int rotate;
  int pdl;
  int TPS;           // tiles per ring batch (capacity)
  int S;             // ring depth (batches)
  int pre_stages;    // batches issued before the compute warps' x / parameter loads are out
  int params_first;  // the first batches wait until the rotation-parameter loads are issued
  int l2_batches;    // stages >= 1: batches prefetched into L2 at the stage boundary
  int xfirst;        // stages >= 1: the ring refill waits until the compute warps' x loads are out
  int nobar;         // experiments only (debug builds): skip the grid-barrier waits
  int n_stages;
  uint32_t* gbar;    // grid barrier words: [0] epoch, [16 ..) one flag per CTA (workspace, zero before first use)
  uint32_t slot_bytes, sc_off, z_off;
  uint32_t off_xp, off_xs, off_scr, off_part, off_recv, off_bar, off_ring, smem_total;
  Gemv1Stage st[MS];
};
using Gemv1Args = Gemv1ArgsT<CHAIN_MAX_STAGES>;

struct Gemv1Config {
  int CL, grid, NW, BT;
  Gemv1Args a;
};

constexpr int PARO_P2P_MAX_WORLD = 8;
// The one-launch B = 1 kernel (gemv1_b1.cu; the round-1 design): B = 1 single launches only.
struct B1Linear {
  const uint8_t* codes;
  const uint8_t* scales;
  const uint8_t* zeros;
  const float2* rot_cs;
  const uchar2* rot_idx;
  const float* svec;
  const float* bias;
  void* y;  // [B][N]
  const uint8_t* xq;  // unused (B = 1)
  const int2* xqs;    // unused (B = 1)
  int N, L;
  int cta_begin, rb_base, rb_extra;
};
struct B1Args {
  const void* x;  // [1][K] fp16 / bf16
  int x_bf16;
  int B;
  int n_lin;
  B1Linear lin[GEMV_MAX_LIN];
  int y_dtype;
  int K, G;
  int rotate;
  int pdl;
  int TPS, S, pre_stages, params_first, atom, R_max, RRmax;
  uint32_t slot_bytes, sc_off, z_off;
  uint32_t off_xp, off_xs, off_scr, off_part, off_recv, off_bar, off_ring, smem_total;
  // NVLink-native all-gather (paro_linear_allgather_p2p): the epilogue stores every y value into
  // each rank's y_full (peer pointers over NVLink) at columns y_col0 + n of rows of length y_ld, and
  // the last CTA to finish releases flag[rank] = epoch + 1 on every rank (system scope)
  int p2p, world, rank;
  int64_t y_ld, y_col0;
  void* peer_y[PARO_P2P_MAX_WORLD];
  uint32_t* peer_flags[PARO_P2P_MAX_WORLD];
  uint32_t* done_ctr;  // local: CTAs finished (the last one resets it)
  int tl_slot;         // PARO_TIMELINE builds: launch slot of the per-CTA timeline
  const uint32_t* epoch;  // local: exchanges completed so far (advanced by the wait kernel)
  // cross-cluster K split (KS > 1, one linear): cluster c takes the K slice c % KS of the row range
  // c / KS; its row sums go to ks_part[slice][n] and the last of the KS clusters to arrive (counter
  // ks_ctr[row range * CL + rank], reset by that CTA) adds the KS slices in a fixed order
  int KS;
  float* ks_part;
  uint32_t* ks_ctr;
};
struct B1Config {
  int CL, grid, NW, BT;
  B1Args a;
};
// ks_part / ks_ctr: the K-split workspace (NULL: no split)
bool plan_gemv1_b1(int B, int n_lin, const int64_t* Ns, int64_t K, int rotate, float* ks_part, uint32_t* ks_ctr,
                   B1Config* cfg, const char** why);
// waits until every rank's flag reached this rank's epoch + 1, then advances the epoch
cudaError_t launch_p2p_wait(uint32_t* flags, uint32_t* epoch, int world, int pdl, cudaStream_t st);
cudaError_t launch_gemv1_b1(const B1Config& cfg, cudaStream_t st);
// cross-cluster K split of a B = 1 launch: slices (1 = none) and the workspace bytes it needs
// (KS x N fp32 row sums); its arrival counters are the KS_CTR_BYTES after s in the packed svec
// buffer (zeroed by paro_pack, left zero by every call)
constexpr size_t KS_CTR_BYTES = 4096;
int b1_ks_slices(int n_lin, const int64_t* Ns, int64_t K);
size_t b1_ks_bytes(int KS, int64_t N);

bool gemv1_enabled();
// B > 1: bytes of pre-transformed activations per linear (digits + per-group sums / scales)
constexpr size_t GEMV1_XQ_GROUP_BYTES = 4096;  // x' bytes reserved per group in the workspace
size_t gemv1_xq_bytes(int B, int64_t K);
// transform pre-kernel of stage 0 (B > 1)
cudaError_t launch_gemv1_xform(const Gemv1Config& cfg, cudaStream_t st);
// Plan a chain: n_stages stages, stage s with n_lin[s] linears of widths Ns[s][i] sharing K[s].
bool plan_gemv1_chain(int B, int n_stages, const int* n_lin, const int64_t (*Ns)[GEMV_MAX_LIN], const int64_t* K,
                      int rotate, int tcgen05, Gemv1Config* cfg, const char** why);
bool plan_gemv1(int B, int n_lin, const int64_t* Ns, int64_t K, int rotate, int tcgen05, Gemv1Config* cfg,
                const char** why);
cudaError_t launch_gemv1(const Gemv1Config& cfg, cudaStream_t st);

// ---------------------------------------------------------------- activation transform (prefill pre-stage)
cudaError_t launch_transform(const void* x, int x_bf16, int64_t B, int64_t K, int L, const float* svec,
                             const float2* rot_cs, const uchar2* rot_idx, int rotate, void* x_out, int pdl,
                             int prefill_order, cudaStream_t st);

// 2-D fp16 tensor map, 128-byte swizzle, box box_inner x box_outer (prefill.cu)
bool make_tmap_2d_f16_sw128(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint32_t box_inner,
                            uint32_t box_outer);
// dense form for many tokens (prefill): M_g rows built by transform_kernel into mrows_ws
// (transform_dense_ws_bytes(K)), then x' = M_g x on the tensor cores
constexpr int64_t DENSE_XFORM_MIN_TOKENS = 64;
size_t transform_dense_ws_bytes(int64_t K);
cudaError_t launch_transform_dense(const void* x, int x_bf16, int64_t B, int64_t K, int L, const float* svec,
                                   const float2* rot_cs, const uchar2* rot_idx, void* x_out, void* mrows_ws, int pdl,
                                   int prefill_order, cudaStream_t st);

// SM-driven 16-byte copy (device or pinned host memory on either side), PDL-capable
cudaError_t launch_copy16(void* dst, const void* src, size_t bytes, int pdl, cudaStream_t st);

// ---------------------------------------------------------------- on-the-fly transform preparation
cudaError_t launch_prepare_transform(const float* theta, const int16_t* pairs, int G, int L, int P, float2* rot_cs,
                                     uchar2* rot_idx, cudaStream_t st);

// ---------------------------------------------------------------- fast Walsh-Hadamard transform (hadamard.cu)
// y (fp16) = scale * H_n diag(signs) x per token; n in {256, ..., 16384}; signs may be NULL
cudaError_t launch_fwht(const void* x, int x_bf16, int64_t T, int64_t n, const float* signs, float scale, void* y,
                        cudaStream_t st);

// ---------------------------------------------------------------- misc
cudaError_t launch_unpack(const uint8_t* codes, const uint8_t* scales, const uint8_t* zeros, int64_t N, int64_t K,
                          uint8_t* codes_u8, uint8_t* scales_f16, uint8_t* zeros_u8, cudaStream_t st);
cudaError_t launch_permute_gather(const void* src, void* dst, int world, int64_t B, int64_t Ns, int elem_bytes,
                                  cudaStream_t st);

// ---------------------------------------------------------------- prefill GEMM (tcgen05)
bool prefill_supported(int64_t B, int64_t N, int64_t K);
cudaError_t launch_prefill_gemm(const void* xq /*fp16 [B][K]*/, int64_t B, const uint8_t* codes, const uint8_t* scales,
                                const uint8_t* zeros, const float* bias, void* y, int y_dtype, int64_t N, int64_t K,
                                int pdl, cudaStream_t st);

// per-device host caches (misc.cu): keyed by the current device, thread-safe
int device_sm_count();
int device_smem_optin();
cudaError_t ensure_smem_attr(const void* fn, int bytes);  // MaxDynamicSharedMemorySize >= bytes on this device
int cached_device_int(const void* fn, int a, int b, int c, int (*compute)(const void*, int, int, int));

}  // namespace paro
