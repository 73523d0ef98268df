/*
 * paro.h -- C ABI of the B200 (sm_100a) ParoQuant hot path.
 *
 * ParoQuant (arXiv 2511.10645): scaled pairwise rotation + group-wise INT4
 * weight-only linear.  Paper text: /root/reference/PAPER.md (cited as PAPER.md:L).
 *
 *   y = (X T^{-1}) Q(T W)^T + b            Eq. 2
 *   T = (prod_{t=1..L} R(P_t, Theta_t)) diag(alpha)   Eq. 8
 *   Q = group-wise RTN, group g = 128      Eq. 1, Fig. 2
 *
 * Conventions:
 *   - W is the PyTorch nn.Linear.weight layout [N, K] row-major (N = D_out,
 *     K = D_in; the paper writes W in R^{D_in x D_out}).
 *   - s is the ACTIVATION multiplier, s = 1/alpha.  The weights get w/s, the
 *     activations s*x (Eq. 2 puts T on W and T^{-1} on X).
 *   - pairs are group-local, 0-based (i, j) with i < j < g, int16, shape
 *     [K/g, L, P, 2]; (-1, -1) marks an absent slot at ANY position (a short
 *     rotation).  theta is fp32 radians, shape [K/g, L, P].
 *   - Rotations are applied scale-first, then t = 1..L ("applied sequentially
 *     after channel-wise scaling"), with the SAME +theta on both
 *     sides: w_n <- R diag(alpha) w_n and x <- R diag(s) x (Eq. 5, PAPER.md:133-138,
 *     re-expressed for column vectors).
 *
 * Threading / ownership:
 *   - The caller owns every device buffer (it allocates the packed buffers after
 *     paro_pack_sizes, and the workspace after paro_linear_workspace).
 *   - The library keeps no pointers across calls.  paro_linear and
 *     paro_transform_activations allocate nothing and never synchronise; they
 *     enqueue on the caller's stream (a cudaStream_t passed as void*).
 *   - Errors are returned as paro_status; a human-readable message for the
 *     calling thread is available from paro_last_error().
 *   - Pointers marked "device" must be CUDA device (or managed) pointers of the
 *     current device; "host" pointers are plain CPU memory.
 */
#ifndef PARO_H_
#define PARO_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PARO_GROUP 128       /* g: quantisation group = rotation group */
#define PARO_MAX_ROT 8       /* L: "8 independent rotations"; L in [0, 8] (Table 6: 0,2,4,8) */
#define PARO_SLOTS 64        /* g/2: max pairs per independent rotation */
#define PARO_BITS 4          /* INT4 */

typedef enum {
  PARO_OK = 0,
  PARO_ERR_INVALID_ARGUMENT = 1, /* bad size, NULL/misaligned pointer, s<=0, non-finite, fp16 scale overflow */
  PARO_ERR_SHAPE = 2,            /* dimension mismatch between arguments */
  PARO_ERR_PAIRS = 3,            /* pairs violate Definition 1 or i<j<g / no cross-rotation repeat */
  PARO_ERR_UNSUPPORTED = 4,      /* K % 128 != 0, group != 128, n_rot > 8, dtype not supported */
  PARO_ERR_CUDA = 5,             /* CUDA runtime error (message in paro_last_error) */
  PARO_ERR_NCCL = 6              /* NCCL error or libnccl.so.2 not loadable */
} paro_status;

typedef enum { PARO_F16 = 0, PARO_BF16 = 1, PARO_F32 = 2 } paro_dtype;

/* Byte sizes of the packed buffers of one linear layer (all device buffers,
 * each must be 16-byte aligned).  Layout (private to the kernels; tests read it
 * only through paro_unpack_logical).  The weight is stored in TILES of 32 output rows x
 * one 128-channel group, tile T = (n / 32) * G + gamma (G = K/128, NB = ceil(N/32) row
 * blocks; rows >= N of the last block are zero):
 *   codes  : NB*G*2048   INT4 codes; row r of a tile is 64 bytes at r*64 whose nibbles hold
 *                        the group's channels in the order the decode kernel's mma.sync
 *                        fragments need (tile_k() in csrc/tile_layout.cuh).
 *   scales : NB*G*64     fp16 group scales S, 32 per tile (rows r, r+8, r+16, r+24 adjacent).
 *   zeros  : NB*G*16     uint4 zero points, 32 per tile (16-bit word r: rows r, r+8, r+16, r+24).
 *   rot_cs : G*L*64*8    fp32 (cos theta, sin theta) per (group, rotation, slot), stored as
 *                        records [G][L][32][2] (slot = lane + 32*s), the slots of each rotation
 *                        reordered and oriented so every shared-memory gather/scatter of the
 *                        runtime transform is bank-conflict free.
 *   rot_idx: G*L*64*2    u8 (i, j) per slot in the same order.
 *   svec   : K*4 + 4096  fp32 s, then the arrival counters of the long-K decode split
 *                        (zeroed by paro_pack; every call leaves them zero, so calls that use
 *                        the same packed linear must be stream-ordered).
 * Weight bytes are N*K/2 + N*G*2 + N*G/2 (0.5195 B/weight) when N % 32 == 0. */
typedef struct {
  size_t codes, scales, zeros, rot_cs, rot_idx, svec;
} paro_packed_sizes;

typedef struct {
  void *codes, *scales, *zeros, *rot_cs, *rot_idx, *svec; /* caller-owned device buffers */
  int64_t N, K;                                           /* output / input channels */
  int32_t group;                                          /* must be 128 */
  int32_t n_rot;                                          /* L in [0, 8] */
} paro_packed;

/* Flags for paro_linear / paro_linear_allgather. */
#define PARO_LINEAR_NO_ROTATION 0x1u /* u = x: skip s and the rotations (plain W4A16; rotation-overhead baseline only) */
#define PARO_LINEAR_PDL 0x2u         /* launch with programmatic dependent launch: weight prefetch may start before
                                        the previous kernel on the stream finishes (weights must not be written by it) */
#define PARO_LINEAR_FORCE_GEMV 0x4u  /* force the decode GEMV kernel for any B (tiles of <= 8 tokens) */
#define PARO_LINEAR_FORCE_GEMM 0x8u  /* force the prefill (tcgen05) path for any B */
#define PARO_LINEAR_TCGEN05 0x10u    /* decode, 2..16 tokens: tiles on the tcgen05 tensor cores (tcgen05.mma
                                        kind::i8, A = u8 codes in TMEM, B = s8 x' digits) instead of the
                                        warp-level mma.sync engine (the default: measured faster) */

/* Sizes of the packed buffers for an [N, K] weight with group size `group`
 * (must be 128) and n_rot rotations (0..8).  Returns PARO_ERR_UNSUPPORTED for
 * K % 128 != 0, group != 128 or n_rot > 8; PARO_ERR_INVALID_ARGUMENT for N, K <= 0
 * or out == NULL. */
paro_status paro_pack_sizes(int64_t N, int64_t K, int32_t group, int32_t n_rot, paro_packed_sizes* out);

/* paro_pack: fold T into W and RTN-quantise ("We then quantize TW instead of W").
 *   W      device fp16 [N, K]
 *   s      device fp32 [K]            activation multiplier s = 1/alpha, finite, > 0
 *   theta  device fp32 [K/128, n_rot, n_pairs]
 *   pairs  device int16 [K/128, n_rot, n_pairs, 2]
 *   n_pairs P in [1, 64]; ignored when n_rot == 0 (theta/pairs may then be NULL)
 *   out    host struct whose buffer pointers the caller filled (sizes from paro_pack_sizes);
 *          the call sets out->N, K, group, n_rot.
 * Per weight row w_n and group gamma (fp64 throughout, each product/sum rounded
 * separately, no FMA):  v = w/s; for t = 1..L, each pair (i, j):
 *   v_i <- cos*v_i - sin*v_j,  v_j <- sin*v_i + cos*v_j      (Eq. 4)
 * then Eq. 1 on the 128 values: S = fp16_rne((max-min)/15) floored at 2^-24,
 * z = clamp(-rint(min/S), 0, 15), q = clamp(rint(v/S) + z, 0, 15) (round half even).
 * cos/sin are evaluated on the host in fp64 with the C library (Q6).
 * Synchronous: copies s/theta/pairs to the host to validate them (Definition 1,
 * i<j<128, no pair repeated across the rotations of a group, s > 0 finite),
 * allocates one temporary of K/128*n_rot*64*16 + 64 bytes with cudaMallocAsync,
 * and returns after the kernel finished.  Errors: PARO_ERR_PAIRS,
 * PARO_ERR_INVALID_ARGUMENT (also for non-finite W or an fp16 scale overflow),
 * PARO_ERR_UNSUPPORTED, PARO_ERR_CUDA. */
paro_status paro_pack(const void* W, const float* s, const float* theta, const int16_t* pairs, int64_t N,
                      int64_t K, int32_t group, int32_t n_rot, int32_t n_pairs, paro_packed* out, void* stream);

/* Workspace bytes paro_linear needs for this call shape.  `on_the_fly` != 0 when paro_linear
 * will be given s/theta/pairs pointers.  Decode with 2..16 tokens needs (G (B'/4) 1024 +
 * G B' 8) bytes (G = K/128, B' = B rounded up to 4, 8 or 16) for the pre-transformed
 * activations.  B = 1 with the packed transform needs 0 bytes, except for a long-K linear with a
 * long weight stream (>= 64 MB, e.g. LLaMA-3-70B down_proj), whose K range is split over
 * KS thread-block clusters: KS x N fp32 row sums (fully written before they are read; no
 * initialisation).  A workspace serves one stream at a time. */
size_t paro_linear_workspace(int64_t B, int64_t N, int64_t K, int32_t n_rot, int32_t n_pairs, int32_t on_the_fly,
                             uint32_t flags);

/* paro_linear: y = (T^{-1} x) . dequant(Q)^T + bias for every token (Eq. 2).
 *   x       device [B, K] fp16 or bf16 (x_dtype), row-major
 *   packed  host struct from paro_pack (device buffers inside)
 *   s, theta, pairs  NULL: use the transform captured in `packed` (normal use).
 *           Non-NULL (all three, device, shapes as in paro_pack with n_pairs):
 *           the transform is prepared on the fly on the GPU (fp32 sincos) into the
 *           workspace; NOT validated -- the caller guarantees Definition 1.
 *   bias    device fp32 [N] or NULL
 *   y       device [B, N] (y_dtype fp16, bf16 or fp32), row-major
 *   flags   PARO_LINEAR_*
 * Decode (B <= 16): B = 1: one fused kernel -- the scale + L rotations are applied to
 * the activation while it is staged in shared memory (never written to HBM), the
 * packed INT4 stream is bulk-copied (TMA engine) into a shared-memory ring and
 * multiplied on the integer tensor cores (x' as 16-bit fixed point per group), exact
 * int32 per (row, group), fp32 accumulate.  B = 2..16: the transform of all tokens runs
 * once in a small kernel into the workspace (x' digits, a few KB per group), then the
 * same GEMV (or, for some widths at B <= 4, a kernel with a cluster-shared in-kernel
 * transform).  Prefill (B > 16): activation
 * transform into an fp16 workspace, then a tcgen05/TMEM GEMM with an in-kernel
 * INT4 -> fp16 dequant producer.
 * Asynchronous, no allocation.  Errors: PARO_ERR_SHAPE (packed vs call), PARO_ERR_INVALID_ARGUMENT
 * (NULL/misaligned pointers, B <= 0, workspace too small), PARO_ERR_UNSUPPORTED (dtypes), PARO_ERR_CUDA.
 * Precision: x' and dequantised weights are never rounded to bf16; |s*x| and |x'| must be < 65504. */
paro_status paro_linear(const void* x, paro_dtype x_dtype, int64_t B, const paro_packed* packed, const float* s,
                        const float* theta, const int16_t* pairs, int32_t n_pairs, const float* bias, void* y,
                        paro_dtype y_dtype, uint32_t flags, void* workspace, size_t workspace_bytes, void* stream);

/* paro_linear_multi: n (1..4) linears that read the SAME activation x (e.g. q/k/v, or
 * gate/up), each with its own transform (one (s, theta, pairs) per linear, Alg. A2,
 * PAPER.md:576-586): y[i] = (T_i^{-1} x) . dequant(Q_i)^T + bias[i].  In decode (B <= 16)
 * all linears run in ONE kernel launch (the clusters of the grid are split over the
 * linears in proportion to their rows), which removes the per-launch prologue of the
 * others; prefill runs one GEMM per linear.  packed, bias (NULL or array of n, entries
 * may be NULL) and y (array of n device [B, N_i]) are host arrays.  All packed[i].K must
 * be equal.  Workspace: n times paro_linear_workspace of the largest linear.  Errors as
 * paro_linear. */
paro_status paro_linear_multi(const void* x, paro_dtype x_dtype, int64_t B, int32_t n, const paro_packed* packed,
                              const float* const* bias, void* const* y, paro_dtype y_dtype, uint32_t flags,
                              void* workspace, size_t workspace_bytes, void* stream);

/* ---- persistent decode chain (fused multi-linear launches, chained) ----
 * A chain is a sequence of decode stages; stage s computes, like paro_linear_multi,
 * y[i] = (T_i^{-1} x) . dequant(Q_i)^T + bias[i] for its n (1..4) linears sharing one x.
 * Stages run IN ORDER with stream semantics: stage s + 1 sees every y stored by stages
 * <= s, so its x may be (a view of) an earlier stage's y (e.g. the down projection reading
 * the up projection's output, or the next layer's q/k/v reading a residual stream the
 * caller's kernels do not touch in between).  Up to 16 stages run in ONE persistent kernel
 * launch: one wave of CTAs, a grid-wide barrier between stages, and the packed weights of
 * all stages streamed back to back through each CTA's shared-memory ring (the weights never
 * depend on earlier stages), so the HBM stream does not stop at stage boundaries; longer
 * chains run as several such launches.  Same arithmetic, layout and precision as
 * paro_linear (Eq. 1, 2, 5, 8).
 *   stages   host array of n_stages; each entry's packed / bias / y are host arrays of n
 *            (bias may be NULL, its entries may be NULL); x and y[i] device, 16-B aligned.
 *            All linears of a stage share K; x is [B][K] of x_dtype, y[i] [B][N_i] of y_dtype.
 *   B        1..16 tokens (decode).
 *   flags    PARO_LINEAR_PDL (the first launch overlaps the previous kernel's tail; the
 *            packed weights must not be written by it), PARO_LINEAR_NO_ROTATION.
 *   workspace  >= paro_linear_chain_workspace(...) bytes, device, 16-B aligned.  Its first
 *            8192 bytes hold the grid-barrier words (a launch epoch and one arrival flag per
 *            CTA): they must be ZERO before the first call (e.g. one cudaMemsetAsync at
 *            allocation); every call advances the epoch, so they never need resetting.  A
 *            workspace serves one stream at a time (calls on it must be stream-ordered).
 * A stage's x must not be written by a LATER stage of the same chain (it is read after the
 * earlier stages only).  Asynchronous, no allocation.  Errors: as paro_linear_multi, plus
 * PARO_ERR_UNSUPPORTED for B > 16. */
typedef struct {
  const void* x;
  int32_t n;
  const paro_packed* packed;
  const float* const* bias;
  void* const* y;
} paro_chain_stage;
size_t paro_linear_chain_workspace(int64_t B, int32_t n_stages, const paro_chain_stage* stages);
paro_status paro_linear_chain(int32_t n_stages, const paro_chain_stage* stages, paro_dtype x_dtype, int64_t B,
                              paro_dtype y_dtype, uint32_t flags, void* workspace, size_t workspace_bytes,
                              void* stream);

/* paro_transform_activations: x' = R_L ... R_1 diag(s) x for every token (the
 * activation side of Eq. 2 / Eq. 5), written as fp16 [B, K] (x_out, device).
 * Uses the transform captured in `packed` (its codes/scales/zeros are not read).
 * Used by the prefill path and exported for tests / the rotation microbenchmark
 * (fig:kernel-speedup).  Asynchronous. */
paro_status paro_transform_activations(const void* x, paro_dtype x_dtype, int64_t B, const paro_packed* packed,
                                       void* x_out, void* stream);

/* paro_transform_activations_dense: the same x' as paro_transform_activations,
 * computed as a dense per-group contraction: per call, M_g = R_L ... R_1 diag(s_g)
 * (128 x 128, the linear map Eq. 5 defines for one group) is
 * built by the Givens kernel applied to the 128 unit vectors and rounded to fp16 into
 * `workspace` (device, >= paro_transform_dense_workspace(K) bytes, 16-byte aligned,
 * caller-owned scratch), then x'_g = M_g x_g for every token on the tensor cores (fp16
 * operands, fp32 accumulation in TMEM, fp16 out).  Results differ from the Givens kernel by
 * the fp16 rounding of M (relative ~2^-11).  The prefill path uses this form for
 * B >= 64 fp16 tokens (bf16 x takes the Givens kernel).  x, x_out 16-byte aligned;
 * fp16 x only (PARO_ERR_UNSUPPORTED otherwise).  Asynchronous. */
size_t paro_transform_dense_workspace(int64_t K);
paro_status paro_transform_activations_dense(const void* x, paro_dtype x_dtype, int64_t B, const paro_packed* packed,
                                             void* x_out, void* workspace, size_t workspace_bytes, void* stream);

/* Test-only: expand the packed weight to logical arrays (device):
 * codes u8 [N, K], scales fp16 [N, K/128], zeros u8 [N, K/128].  Asynchronous. */
paro_status paro_unpack_logical(const paro_packed* packed, void* codes_u8, void* scales_f16, void* zeros_u8,
                                void* stream);

/* paro_copy: dst <- src (bytes, a multiple of 16; both pointers 16-byte aligned), copied by the
 * SMs (one 16-byte load/store per thread).  Either side may be device memory or pinned host memory
 * (cudaHostAlloc / torch pin_memory; unified addressing), so a serving loop moves a step's tokens
 * in and its outputs out through PCIe without a DMA-engine copy node between its kernels.  With
 * PARO_LINEAR_PDL the copy is a programmatic dependent of the previous kernel on the stream (reads
 * src after that kernel completed) and lets the next kernel launch early.  Asynchronous; host
 * memory written by it is complete once the stream work is complete.  Errors:
 * PARO_ERR_INVALID_ARGUMENT (NULL / misaligned), PARO_ERR_CUDA. */
paro_status paro_copy(void* dst, const void* src, size_t bytes, uint32_t flags, void* stream);

/* ---- fast Walsh-Hadamard transform (comparison transform) ----
 * The transform the paper's kernel experiment compares against (fig:kernel-speedup,
 * PAPER.md:200-209): per token, y = scale * H_n diag(signs) x with H_n the
 * Sylvester Hadamard matrix, H[i, j] = (-1)^popcount(i & j) (the unnormalised butterfly;
 * scale = 1/sqrt(n) and random +-1 signs give the randomised orthogonal variant).
 *   x      device [T, n] fp16 / bf16, 16-B aligned       T  tokens (> 0)
 *   n      power of two in [256, 16384]                   signs  device fp32 [n] or NULL (all +1)
 *   y      device [T, n] fp16 (fp32 arithmetic, one rounding)
 * Asynchronous on `stream`, no allocation.  Errors: PARO_ERR_INVALID_ARGUMENT (NULL /
 * misaligned pointers, T <= 0), PARO_ERR_UNSUPPORTED (n, dtype), PARO_ERR_CUDA. */
paro_status paro_fwht(const void* x, paro_dtype x_dtype, int64_t T, int64_t n, const float* signs, float scale,
                      void* y, void* stream);

/* ---- Alg. A1: selection of independent channel pairs ----
 * PAPER.md:509-553 (Alg. A1): for each of `n_groups` groups of g
 * channels, shuffle all g(g-1)/2 pairs (i < j) once, then for rotation r = 1..n_rot
 * greedily take the next pairs of the shuffled list whose channels are unused in this
 * rotation and which no earlier rotation took, up to n_pairs; a rotation may run short
 * (its remaining slots are (-1, -1)).  Every output rotation satisfies Definition 1
 * and no pair repeats across the rotations of a group, so the result
 * is valid `pairs` input for paro_pack.
 * Shuffle (Q20): xoshiro256** whose state for group gamma is
 * outputs 4 gamma .. 4 gamma + 3 of SplitMix64 seeded with `seed`; Fisher-Yates from the
 * last element down, j = uniform [0, i] by rejection of draws below 2^64 mod (i + 1).
 *   pairs_out : HOST int16 [n_groups][n_rot][n_pairs][2], caller-owned, fully written.
 * Runs on the calling thread (host code, offline); no CUDA call.
 * Errors: PARO_ERR_INVALID_ARGUMENT unless 2 <= g <= 4096, n_rot >= 1,
 *         1 <= n_pairs <= g/2, n_groups >= 0 and pairs_out != NULL (when n_groups > 0). */
paro_status paro_select_pairs(int64_t n_groups, int32_t g, int32_t n_rot, int32_t n_pairs, uint64_t seed,
                              int16_t* pairs_out);

/* ---- output-channel (N) sharding over NVLink ----
 * Rank r of G owns rows [r*N/G, (r+1)*N/G) of W, packed with paro_pack on that
 * row slice (identical, bitwise, to the same rows of the full pack).  Every rank
 * holds the full x, applies the (cheap) transform locally, runs the GEMV on its
 * shard, and an NCCL all-gather of y runs on the same stream.
 * libnccl.so.2 is loaded at first use with dlopen (the copy already mapped by the
 * process, e.g. PyTorch's, is reused). */
#define PARO_NCCL_UNIQUE_ID_BYTES 128

/* Fill `uid` (host, 128 bytes) with a fresh ncclUniqueId.  Call on one rank and
 * broadcast the bytes (e.g. over a torch.distributed process group). */
paro_status paro_comm_unique_id(void* uid);
/* Create an NCCL communicator for (rank, world) from the broadcast uid; *comm
 * receives an opaque handle (an ncclComm_t).  Collective over all ranks. */
paro_status paro_comm_init(const void* uid, int32_t rank, int32_t world, void** comm);
paro_status paro_comm_destroy(void* comm);
/* Asynchronous NCCL errors (a failed peer, a broken link) detected since the last call:
 * PARO_OK, or PARO_ERR_NCCL with the NCCL message in paro_last_error().  Also checked by
 * paro_linear_allgather before and after it enqueues the collective. */
paro_status paro_comm_check(void* comm);

/* Sharded linear: packed_shard holds this rank's N/world rows; y_full is device
 * [B, N] (N = packed_shard->N * world) in y_dtype.  workspace must hold
 * paro_linear_allgather_workspace(...) bytes.  Errors as paro_linear, plus
 * PARO_ERR_NCCL. */
size_t paro_linear_allgather_workspace(int64_t B, int64_t N_shard, int64_t K, int32_t world, paro_dtype y_dtype,
                                       uint32_t flags);
paro_status paro_linear_allgather(const void* x, paro_dtype x_dtype, int64_t B, const paro_packed* packed_shard,
                                  const float* bias_shard, void* y_full, paro_dtype y_dtype, uint32_t flags,
                                  void* workspace, size_t workspace_bytes, void* comm, int32_t rank, int32_t world,
                                  void* stream);

/* Message of the last error on the calling thread ("" if none). */
/* ---- NVLink-native all-gather of y ----
 * The N-sharded decode linear without NCCL: rank r's GEMV epilogue stores each of its y values
 * straight into EVERY rank's y_full (P2P stores over NVLink / NVSwitch through CUDA IPC peer
 * pointers) at columns [r Ns, (r+1) Ns), and the last of its CTAs releases flag[r] on every rank
 * (system scope); a one-thread wait kernel then holds the stream until all ranks' flags arrived.
 * Per-rank buffer (paro_p2p_buffer_bytes, zero before first use, never reset): y_full [1][N_full]
 * of y_dtype, then the flags / epoch / CTA counter.  Epochs advance once per call on every rank, so
 * calls must be matched across ranks (same order), and the buffers may be captured in CUDA graphs.
 *   peer_bufs  host array [world]: the device pointer of every rank's buffer as seen from this
 *              process (own rank: its local pointer; others: paro_ipc_open_handle)
 *   B          must be 1 (decode).  Errors as paro_linear_allgather; PARO_ERR_UNSUPPORTED for B != 1.
 * The result is this rank's y_full (its own buffer) once the call's kernels ran on `stream`. */
size_t paro_p2p_buffer_bytes(int64_t B, int64_t N_full, paro_dtype y_dtype, int32_t world);
paro_status paro_ipc_get_handle(const void* dev_ptr, void* handle /* 64 bytes, host */);
paro_status paro_ipc_open_handle(const void* handle, void** dev_ptr);
paro_status paro_ipc_close_handle(void* dev_ptr);
paro_status paro_linear_allgather_p2p(const void* x, paro_dtype x_dtype, int64_t B, const paro_packed* packed_shard,
                                      const float* bias_shard, paro_dtype y_dtype, uint32_t flags,
                                      void* const* peer_bufs, int32_t rank, int32_t world, void* stream);

const char* paro_last_error(void);
/* Library version string. */
const char* paro_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PARO_H_ */
