"""ParoQuant CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this module.  The product path
(``paper_2511_10645_b200``) never imports, links or executes it, and it shares no
code with the CUDA path (no kernels, headers, helpers, tables or constants).

Plain, slow, obviously-correct fp64 numpy, written step by step from the paper
(arXiv 2511.10645, text in PAPER.md) in the paper's order and notation.  Each
function cites the passage it follows.  Readings where the paper is silent or
ambiguous are the SURVEY.md 8(c) readings Q1..Q19, listed in DESIGN.md.

Conventions:
  * W is PyTorch ``nn.Linear.weight`` layout [N, K] (paper: W in R^{D_in x D_out},
    PAPER.md:62 -- the transpose).  Row n of W is the K-vector w_n.
  * s is the activation-side multiplier, s = 1/alpha (Eq. 8's alpha scales W,
    PAPER.md:178; Eq. 2 puts the inverse on X).
  * pairs are group-local, 0-based, i < j, (-1,-1) padding.

Parity pins: every function here is pinned by tests/test_oracle_*.py against
closed forms, brute force, worked examples and library routines (see DESIGN.md
"Oracle pins").  The only part without an independent pin at realistic shapes is
the composition at full size, which the paper never prints ("parity unpinned" for
realistic-shape VALUES: PAPER.md prints no numeric pack/linear outputs; the
figures are .pgf not included).
"""
from __future__ import annotations

import math

import numpy as np


class OracleError(ValueError):
    """kind in {"invalid_argument", "shape", "pairs", "unsupported"} (SURVEY.md 8(b) errors)."""

    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


# --------------------------------------------------------------------------------------
# Validation: Definition 1 (independent pairs) and the TransformBundle invariants
# --------------------------------------------------------------------------------------
def validate_transform(K: int, s: np.ndarray, theta: np.ndarray, pairs: np.ndarray, g: int = 128) -> None:
    """Def. 1: within one rotation every channel appears in at most
    one pair.  Plus SPEC.md:213 (i<j<g), SPEC.md:227 (no pair repeated across the
    rotations of a group, Alg. A1's "block pair"), SPEC.md:226 (alpha>0).
    """
    if g < 2 or K <= 0:
        raise OracleError("invalid_argument", "g < 2 or K <= 0")
    if K % g:
        raise OracleError("unsupported", "K % g != 0 (SURVEY.md Q17)")
    G = K // g
    if s.shape != (K,):
        raise OracleError("shape", "s must be [K]")
    if not np.all(np.isfinite(s)) or np.any(s <= 0):
        raise OracleError("invalid_argument", "s must be finite and > 0")
    if pairs.ndim != 4 or pairs.shape[0] != G or pairs.shape[3] != 2:
        raise OracleError("shape", "pairs must be [K/g, L, P, 2]")
    L, P = pairs.shape[1], pairs.shape[2]
    if theta.shape != (G, L, P):
        raise OracleError("shape", "theta must be [K/g, L, P]")
    if P > g // 2:
        raise OracleError("invalid_argument", "P > g/2")
    if not np.all(np.isfinite(theta)):
        raise OracleError("invalid_argument", "theta must be finite")
    for gam in range(G):
        seen_pairs = set()
        for t in range(L):
            used = set()
            for p in range(P):
                i, j = int(pairs[gam, t, p, 0]), int(pairs[gam, t, p, 1])
                if i == -1 and j == -1:
                    continue                                   # padded slot
                if i < 0 or j < 0 or i >= g or j >= g:
                    raise OracleError("pairs", f"index out of range at ({gam},{t},{p})")
                if not i < j:
                    raise OracleError("pairs", f"need i < j at ({gam},{t},{p})")
                if i in used or j in used:                     # Definition 1
                    raise OracleError("pairs", f"channel reused in rotation ({gam},{t})")
                used.add(i)
                used.add(j)
                if (i, j) in seen_pairs:                        # Alg. A1 "block pair"
                    raise OracleError("pairs", f"pair repeated across rotations in group {gam}")
                seen_pairs.add((i, j))


# --------------------------------------------------------------------------------------
# Givens rotations: Eq. 3 / Eq. 4 / Eq. 5 / Def. 2 / Eq. 8
# --------------------------------------------------------------------------------------
def givens_coefficients(theta: np.ndarray):
    """cos(theta), sin(theta) in fp64 from the fp32 angle, via the host C library
    (Python's math.cos/math.sin call libm) -- SURVEY.md Q6."""
    flat = theta.astype(np.float64).ravel()
    c = np.array([math.cos(t) for t in flat], dtype=np.float64).reshape(theta.shape)
    sn = np.array([math.sin(t) for t in flat], dtype=np.float64).reshape(theta.shape)
    return c, sn


def apply_independent_rotations(V: np.ndarray, theta: np.ndarray, pairs: np.ndarray, g: int = 128) -> np.ndarray:
    """Apply R(P_L,Theta_L) ... R(P_1,Theta_1) to the channel axis (axis 0) of V [K, M], in place.

    Eq. 4: for each pair (i, j) with angle theta,
        V[i] <- cos(theta) V[i] - sin(theta) V[j]
        V[j] <- sin(theta) V[i] + cos(theta) V[j]      (both from pre-update values)
    Rotations t = 1..L are applied in order (Eq. 3's G_1-first convention,
    PAPER.md:122).  Within one rotation the pairs are independent
    (Def. 2): they touch disjoint channels, so all pairs of one
    rotation -- in every group, since groups are disjoint too -- are
    updated together.  Each product and each sum is a separately rounded fp64 numpy
    operation (no fused multiply-add).
    """
    K = V.shape[0]
    G = K // g
    L = pairs.shape[1]
    c, sn = givens_coefficients(theta)
    for t in range(L):                                         # rotation t (sequential)
        pr = pairs[:, t]                                       # [G, P, 2]
        valid = pr[..., 0] >= 0                                # skip (-1,-1) slots
        gam = np.broadcast_to(np.arange(G)[:, None], valid.shape)[valid]
        I = gam * g + pr[..., 0][valid].astype(np.int64)
        J = gam * g + pr[..., 1][valid].astype(np.int64)
        ct = c[:, t][valid][:, None]
        st = sn[:, t][valid][:, None]
        a = V[I].copy()                                        # pre-update values
        b = V[J].copy()
        V[I] = (ct * a) - (st * b)
        V[J] = (st * a) + (ct * b)
    return V


def fold(W: np.ndarray, s: np.ndarray, theta: np.ndarray, pairs: np.ndarray, g: int = 128) -> np.ndarray:
    """T(W) of Eq. 8 in the [N, K] layout: for every weight row w_n,
        v_n = R_L ... R_1 diag(alpha) w_n,   alpha = 1/s,
    with the scaling applied FIRST ("The independent rotations are applied
    sequentially after channel-wise scaling").  diag(alpha) w is
    computed as w / s (one correctly-rounded division).
    Returns fp64 [N, K]."""
    V = W.astype(np.float64).T / s.astype(np.float64)[:, None]   # [K, N]: diag(alpha) W^T
    apply_independent_rotations(V, theta, pairs, g)
    return V.T.copy()


def transform_activations(x: np.ndarray, s: np.ndarray, theta: np.ndarray, pairs: np.ndarray,
                          g: int = 128) -> np.ndarray:
    """X T^{-1} of Eq. 2 with T = (prod R_t) diag(alpha) (Eq. 8).

    In column form, for a token x (K-vector): x' = R_L ... R_1 diag(s) x, i.e. the
    SAME rotations with the SAME +theta in the SAME order t = 1..L, after scaling by
    s = 1/alpha.  This is Eq. 5's "reverse the sequence and negate theta"
     re-expressed for column vectors: row-vector X G(-theta_1)...
    G(-theta_m) transposed is G(theta_m)...G(theta_1) x^T (SPEC.md:265's
    "divide column c by alpha at the end" is the reading we reject -- the master
    identity SPEC.md:270 fixes it).  x is [B, K]; returns fp64 [B, K]."""
    U = (x.astype(np.float64) * s.astype(np.float64)[None, :]).T.copy()   # diag(s) x, exact
    apply_independent_rotations(U, theta, pairs, g)
    return U.T.copy()


# --------------------------------------------------------------------------------------
# Eq. 1: RTN linear quantisation, block-wise along the input dimension
# --------------------------------------------------------------------------------------
FP16_MIN_SUBNORMAL = 2.0 ** -24


def rtn_groups(V: np.ndarray, bits: int = 4, g: int = 128):
    """Eq. 1 with one (s, z) per g consecutive input-channel elements
    of each output row:
        s = (max(X) - min(X)) / (2^b - 1),   z = -round(min(X)/s),
        Q = clamp(round(X/s) + z, 0, 2^b - 1).
    Readings: round = half-to-even (Q9); the scale is STORED in fp16 by a
    single round-to-nearest-even from fp64 and floored at 2^-24 (Q8, Q10); z and the
    codes are computed against that stored scale (Q8); z is clamped to [0, 2^b-1]
    (Q11).  V is fp64 [N, K]; returns codes uint8 [N, K], scales fp16 [N, K/g],
    zeros uint8 [N, K/g]."""
    N, K = V.shape
    G = K // g
    qmax = float(2 ** bits - 1)
    Vg = V.reshape(N, G, g)
    mn = Vg.min(axis=2)
    mx = Vg.max(axis=2)
    s64 = (mx - mn) / qmax
    S = s64.astype(np.float16)                                 # one RNE rounding fp64 -> fp16
    if not np.all(np.isfinite(S)):
        raise OracleError("invalid_argument", "fp16 group scale overflows")
    S = np.where(S.astype(np.float64) < FP16_MIN_SUBNORMAL, np.float16(FP16_MIN_SUBNORMAL), S)
    S64 = S.astype(np.float64)
    z = np.clip(-np.rint(mn / S64), 0.0, qmax)
    q = np.clip(np.rint(Vg / S64[:, :, None]) + z[:, :, None], 0.0, qmax)
    return q.reshape(N, K).astype(np.uint8), S, z.astype(np.uint8)


def dequantize(codes: np.ndarray, scales: np.ndarray, zeros: np.ndarray, g: int = 128) -> np.ndarray:
    """v_hat = (q - z) * s (SPEC.md:152, 187 -- the paper omits the inverse map).  fp64 [N, K]."""
    N, K = codes.shape
    G = K // g
    q = codes.reshape(N, G, g).astype(np.float64)
    return ((q - zeros.astype(np.float64)[:, :, None]) * scales.astype(np.float64)[:, :, None]).reshape(N, K)


# --------------------------------------------------------------------------------------
# The two calls of the boundary
# --------------------------------------------------------------------------------------
def oracle_pack(W: np.ndarray, s: np.ndarray, theta: np.ndarray, pairs: np.ndarray, g: int = 128):
    """paro_pack: validate, fold T into W (Eq. 8), then RTN-quantise (Eq. 1).
    "We then quantize TW instead of W"; Q group = rotation group
    (Fig. 2 caption).  Returns dict(codes u8 [N,K], scales f16 [N,G],
    zeros u8 [N,G], V fp64 [N,K] (the folded, unquantised weight))."""
    N, K = W.shape
    if N <= 0:
        raise OracleError("invalid_argument", "N <= 0")
    validate_transform(K, s, theta, pairs, g)
    if not np.all(np.isfinite(W.astype(np.float64))):
        raise OracleError("invalid_argument", "W must be finite")
    V = fold(W, s, theta, pairs, g)
    codes, scales, zeros = rtn_groups(V, 4, g)
    return dict(codes=codes, scales=scales, zeros=zeros, V=V)


def oracle_linear(x: np.ndarray, packed: dict, s: np.ndarray, theta: np.ndarray, pairs: np.ndarray,
                  bias: np.ndarray | None = None, g: int = 128, rotate: bool = True) -> np.ndarray:
    """paro_linear: y = (X T^{-1}) Q(TW)^T + b (Eq. 2), fp64 [B, N].

    x' = transform_activations(x) (Eq. 5 / Eq. 8 inverse); then the group-wise INT4
    dequant-dot  y[b,n] = sum_gamma S[n,gamma] * sum_{k in gamma} (q[n,k] - z[n,gamma]) x'[b,k]
    (a library matmul over the dequantised fp64 weight).  rotate=False gives the
    plain W4A16 dot x . dequant(Q)^T used as the rotation-off timing baseline."""
    xp = transform_activations(x, s, theta, pairs, g) if rotate else x.astype(np.float64)
    Wq = dequantize(packed["codes"], packed["scales"], packed["zeros"], g)
    y = xp @ Wq.T
    if bias is not None:
        y = y + bias.astype(np.float64)[None, :]
    return y


def linear_fp(x: np.ndarray, W: np.ndarray, bias: np.ndarray | None = None) -> np.ndarray:
    """Unquantised Y = X W + b (Eq. 2 left side), fp64 [B, N]."""
    y = x.astype(np.float64) @ W.astype(np.float64).T
    if bias is not None:
        y = y + bias.astype(np.float64)[None, :]
    return y


def materialize(s_group: np.ndarray, theta_group: np.ndarray, pairs_group: np.ndarray) -> np.ndarray:
    """Dense g x g matrix M = R_L ... R_1 diag(alpha) of one group,
    obtained by applying fold's rotation step to the g unit vectors.  Testing aid."""
    g = s_group.shape[0]
    E = np.eye(g, dtype=np.float64) / s_group.astype(np.float64)[:, None]
    apply_independent_rotations(E, theta_group[None], pairs_group[None], g)
    return E


def normwise_error(y: np.ndarray, y_ref: np.ndarray) -> float:
    """max_{b,n}|y - y_ref| / max_{b,n}|y_ref| (normwise infinity)."""
    d = np.max(np.abs(y.astype(np.float64) - y_ref.astype(np.float64)))
    m = np.max(np.abs(y_ref.astype(np.float64)))
    return float(d / m) if m > 0 else float(d)
