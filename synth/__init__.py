"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests, smoke() and bench.py.

This module holds NO ParoQuant arithmetic: no scaling, no Givens rotation, no
quantisation.  It only draws random tensors with the shapes and structure of the
paper's workloads and builds pair lists with the structure of Alg. A1.

Recipe (also in DESIGN.md, "Input recipe"):
  * W  ~ N(0, 0.02^2), fp16, [N, K] (PyTorch nn.Linear layout).  Parity sets add a
    few outlier input channels with gain 50 (SPEC.md:516-528 OutlierModelSpec idea)
    and optionally an all-zero group.
  * x  ~ N(0, 1), fp16 or bf16, [B, K], with 1 % outlier channels x20
    (activation outliers, "outlier channels").
  * s  = exp(U(-0.5, 0.5)), fp32, [K]: the activation-side multiplier s = 1/alpha
    (alpha is initialised at 1 and learned; its learned range is
    unpublished).
  * theta ~ U(-pi, pi), fp32, [G, L, P] (radians, unconstrained).
  * pairs: Alg. A1, group-local 0-based (i, j), i < j,
    int16 [G, L, P, 2], (-1, -1) padding for short rotations.

Random numbers come from numpy's PCG64 ``default_rng(seed)``; SPEC.md:87's
SplitMix64/xoshiro256** is not needed because nothing here must be reproduced
by another language.
"""
from __future__ import annotations

import math

import numpy as np

GROUP = 128      # g
N_ROT = 8        # K in Eq. 8 / Alg. A1
N_PAIRS = 64     # N in Alg. A1 ("up to 64 pairs")


def select_pairs(n_groups: int, g: int = GROUP, n_rot: int = N_ROT, n_pairs: int = N_PAIRS,
                 seed: int = 0) -> np.ndarray:
    """Alg. A1 "Selection of Independent Channel Pairs", run for
    every group independently (Alg. A2 line "for i <- 1 to n: P_i <- SelectPairs(W_i,K,N)",
    PAPER.md:577).  Returns int16 [n_groups, n_rot, n_pairs, 2], 0-based, i < j,
    (-1, -1) where a rotation ran short.

    The algorithm is followed literally -- one shuffle of all g(g-1)/2 pairs per
    group, then per rotation a greedy pass over the shuffled list that skips pairs
    whose channels are already used in this rotation or that were used by an
    earlier rotation -- but the pass is vectorised ACROSS groups (each group has
    its own shuffled list and its own availability state), which changes nothing
    about any single group's result.
    """
    if g < 2 or n_rot < 0 or not (1 <= n_pairs <= g // 2):
        raise ValueError("select_pairs: need g>=2, n_rot>=0, 1<=n_pairs<=g/2")
    rng = np.random.default_rng(seed)
    iu, ju = np.triu_indices(g, k=1)                       # P = {(i,j) | i<j}
    n_all = iu.size
    # P_shuffled, one permutation per group
    perm = np.stack([rng.permutation(n_all) for _ in range(n_groups)]) if n_groups else \
        np.zeros((0, n_all), dtype=np.int64)
    pi = iu[perm]                                          # [G, n_all]
    pj = ju[perm]
    out = np.full((n_groups, n_rot, n_pairs, 2), -1, dtype=np.int16)
    pair_used = np.zeros((n_groups, n_all), dtype=bool)   # matrix A ("block pair")
    gidx = np.arange(n_groups)
    for r in range(n_rot):
        ch_used = np.zeros((n_groups, g), dtype=bool)     # A_rot ("block channels")
        count = np.zeros(n_groups, dtype=np.int64)
        for p in range(n_all):
            if n_groups == 0 or (count >= n_pairs).all():
                break
            i = pi[:, p]
            j = pj[:, p]
            flat = perm[:, p]
            ok = (count < n_pairs) & ~ch_used[gidx, i] & ~ch_used[gidx, j] & ~pair_used[gidx, flat]
            if not ok.any():
                continue
            gs = gidx[ok]
            out[gs, r, count[ok], 0] = i[ok]
            out[gs, r, count[ok], 1] = j[ok]
            ch_used[gs, i[ok]] = True
            ch_used[gs, j[ok]] = True
            pair_used[gs, flat[ok]] = True
            count[ok] += 1
    return out


def make_problem(N: int, K: int, B: int = 1, *, seed: int = 0, g: int = GROUP, n_rot: int = N_ROT,
                 n_pairs: int = N_PAIRS, x_dtype=np.float16, outliers: bool = True,
                 zero_group: bool = False, theta_mode: str = "uniform", s_mode: str = "random",
                 with_bias: bool = False, special_groups: bool = False, x_zero_group: bool = False,
                 x_big: float = 0.0) -> dict:
    """One seeded linear-layer instance: W fp16 [N,K], x [B,K], s fp32 [K],
    theta fp32 [G,L,P], pairs int16 [G,L,P,2], optional bias fp32 [N].

    theta_mode: "uniform" (U(-pi,pi)), "zero", "quarter" (pi/2), "eighth" (pi/4).
    s_mode:     "random" (exp(U(-.5,.5))), "ones".
    special_groups (needs K >= 5 g): group 2 of W all positive, group 3 all negative, group 4
        the constant 0.5, each with theta = 0 in that group (and s = 1 on group 4), so the
        weight the quantiser sees keeps that structure (one-signed / constant groups:
        the zero-point clamp and the scale floor of Eq. 1).
    x_zero_group: x is 0 on every channel of group 0 (an all-zero activation group).
    x_big:      if > 0, one channel per group of x is set to +-x_big (activations near the
        fp16 range; |s x| stays below 65504 for x_big <= 39000).
    """
    if K % g:
        raise ValueError("K must be a multiple of the group size")
    rng = np.random.default_rng(seed + 1_000_003)
    G = K // g
    W = rng.normal(0.0, 0.02, size=(N, K))
    if outliers and K >= 8:
        oc = rng.choice(K, size=min(4, K), replace=False)   # 4 outlier input channels, gain 50
        W[:, oc] *= 50.0
    if zero_group and G >= 2:
        W[:, g:2 * g] = 0.0                                 # one all-zero group
    if special_groups:
        if G < 5:
            raise ValueError("special_groups needs K >= 5 g")
        W[:, 2 * g:3 * g] = np.abs(W[:, 2 * g:3 * g]) + 1e-3     # all positive
        W[:, 3 * g:4 * g] = -np.abs(W[:, 3 * g:4 * g]) - 1e-3    # all negative
        W[:, 4 * g:5 * g] = 0.5                                 # constant nonzero
    W = W.astype(np.float16)
    x = rng.normal(0.0, 1.0, size=(B, K))
    if outliers:
        nx = max(1, K // 100)                               # 1 % outlier channels x20
        xc = rng.choice(K, size=nx, replace=False)
        x[:, xc] *= 20.0
    if x_zero_group:
        x[:, 0:g] = 0.0
    if x_big > 0:
        cols = np.arange(G) * g + rng.integers(0, g, size=G)
        x[:, cols] = x_big * np.where(rng.random((B, G)) < 0.5, -1.0, 1.0)
    if x_dtype == "bf16":
        x = x.astype(np.float32)                            # rounded to bf16 by the caller (torch)
    else:
        x = x.astype(x_dtype)
    if s_mode == "ones":
        s = np.ones(K, dtype=np.float32)
    else:
        s = np.exp(rng.uniform(-0.5, 0.5, size=K)).astype(np.float32)
    if theta_mode == "uniform":
        theta = rng.uniform(-math.pi, math.pi, size=(G, n_rot, n_pairs)).astype(np.float32)
    elif theta_mode == "zero":
        theta = np.zeros((G, n_rot, n_pairs), dtype=np.float32)
    elif theta_mode == "quarter":
        theta = np.full((G, n_rot, n_pairs), math.pi / 2, dtype=np.float32)
    elif theta_mode == "eighth":
        theta = np.full((G, n_rot, n_pairs), math.pi / 4, dtype=np.float32)
    else:
        raise ValueError(theta_mode)
    pairs = select_pairs(G, g=g, n_rot=n_rot, n_pairs=n_pairs, seed=seed)
    theta = np.where(pairs[..., 0] < 0, np.float32(0), theta).astype(np.float32)
    if special_groups:
        theta[2:5] = 0.0
        s[4 * g:5 * g] = 1.0
    bias = rng.normal(0.0, 0.1, size=N).astype(np.float32) if with_bias else None
    return dict(W=W, x=x, s=s, theta=theta, pairs=pairs, bias=bias, N=N, K=K, B=B, g=g, n_rot=n_rot)


def single_pair_problem(N: int = 256, K: int = 256, *, group: int = 1, layer: int = 3,
                        i: int = 5, j: int = 77, theta: float = math.pi / 4, seed: int = 0) -> dict:
    """Every slot padded except ONE active pair (i, j) in one (group, layer): the
    closed-form single-Givens case."""
    p = make_problem(N, K, 1, seed=seed, s_mode="ones", theta_mode="zero")
    pairs = np.full_like(p["pairs"], -1)
    th = np.zeros_like(p["theta"])
    pairs[group, layer, 17] = (i, j)
    th[group, layer, 17] = theta
    p["pairs"], p["theta"] = pairs, th
    return p


def force_short_layers(p: dict, seed: int = 0, frac: float = 0.1) -> dict:
    """Pad random slots (at arbitrary positions) with (-1,-1): rotations shorter than
    64 pairs ("insufficient number of pairs")."""
    rng = np.random.default_rng(seed + 77)
    pairs = p["pairs"].copy()
    theta = p["theta"].copy()
    mask = rng.random(pairs.shape[:3]) < frac
    pairs[mask] = -1
    theta[mask] = 0.0
    q = dict(p)
    q["pairs"], q["theta"] = pairs, theta
    return q


# Shapes of the paper's workloads (BASELINE.json configs)
LLAMA3_8B_DECODE = {            # name: (N, K) in nn.Linear [out, in] layout
    "q_proj": (4096, 4096), "k_proj": (1024, 4096), "v_proj": (1024, 4096), "o_proj": (4096, 4096),
    "gate_proj": (14336, 4096), "up_proj": (14336, 4096), "down_proj": (4096, 14336),
}
QWEN3_4B_LAYER = {
    "q_proj": (4096, 2560), "k_proj": (1024, 2560), "v_proj": (1024, 2560), "o_proj": (2560, 4096),
    "gate_proj": (9728, 2560), "up_proj": (9728, 2560), "down_proj": (2560, 9728),
}
QWEN3_4B_LAYERS = 36
LLAMA3_70B_MLP = {"gate_proj": (28672, 8192), "up_proj": (28672, 8192), "down_proj": (8192, 28672)}
