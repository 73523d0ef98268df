"""Pins of the fp64 oracle against things other than itself (closed forms, worked
examples from the paper/SPEC, brute force on tiny inputs, invariants, an independent
library routine).  CPU only."""
import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle as O
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")))


def dense_givens(g, i, j, theta):
    """Explicit Givens matrix G(i, j, theta) of Eq. 3: rotates rows
    i and j: [G]_{ii}=c, [G]_{ij}=-s, [G]_{ji}=s, [G]_{jj}=c (matrix form of Eq. 4)."""
    G = np.eye(g)
    c, s = np.cos(theta), np.sin(theta)
    G[i, i], G[i, j], G[j, i], G[j, j] = c, -s, s, c
    return G


def dense_transform(alpha, theta, pairs):
    """Brute-force dense T = G_{L,P}...G_{1,1} diag(alpha) for one group, as an explicit
    product of Givens matrices in the paper's order (Eq. 3 + Eq. 8)."""
    g = alpha.shape[0]
    M = np.diag(alpha.astype(np.float64))
    for t in range(pairs.shape[0]):
        for p in range(pairs.shape[1]):
            i, j = int(pairs[t, p, 0]), int(pairs[t, p, 1])
            if i < 0:
                continue
            M = dense_givens(g, i, j, float(theta[t, p])) @ M
    return M


# ------------------------------------------------------------------ fold / rotation pins
def test_theta_zero_is_bitwise_identity():
    """theta=0, alpha=1 is the identity (the paper's initialisation):
    c=1, sn=0 make Eq. 4 exact in floating point."""
    p = synth.make_problem(64, 256, theta_mode="zero", s_mode="ones", seed=3)
    V = O.fold(p["W"], p["s"], p["theta"], p["pairs"])
    assert np.array_equal(V, p["W"].astype(np.float64))


def test_single_pair_closed_form_eighth_turn():
    """One active pair at theta=pi/4: v_i=(w_i-w_j)/sqrt2, v_j=(w_i+w_j)/sqrt2; every
    other channel untouched (Eq. 4 closed form)."""
    p = synth.single_pair_problem(N=32, K=256, group=1, layer=2, i=5, j=77, theta=math.pi / 4)
    V = O.fold(p["W"], p["s"], p["theta"], p["pairs"])
    W = p["W"].astype(np.float64)
    I, J = 128 + 5, 128 + 77
    r2 = math.sqrt(2.0)
    tol = 1e-7 * np.max(np.abs(W))                       # theta is fp32: |fl32(pi/4) - pi/4| < 3e-8
    np.testing.assert_allclose(V[:, I], (W[:, I] - W[:, J]) / r2, rtol=0, atol=tol)
    np.testing.assert_allclose(V[:, J], (W[:, I] + W[:, J]) / r2, rtol=0, atol=tol)
    other = np.ones(256, bool)
    other[[I, J]] = False
    assert np.array_equal(V[:, other], W[:, other])


def test_quarter_turn_orientation():
    """theta=pi/2 -> row_i' = -row_j, row_j' = row_i (catches a swapped
    sign / orientation)."""
    p = synth.single_pair_problem(N=16, K=128, group=0, layer=0, i=3, j=9, theta=math.pi / 2)
    V = O.fold(p["W"], p["s"], p["theta"], p["pairs"])
    W = p["W"].astype(np.float64)
    tol = 1e-7 * np.max(np.abs(W))                       # cos(fl32(pi/2)) = -4.4e-8
    np.testing.assert_allclose(V[:, 3], -W[:, 9], atol=tol)
    np.testing.assert_allclose(V[:, 9], W[:, 3], atol=tol)


def test_spec_2x2_bundle_example():
    """g=2, alpha=(2,1), pair (0,1), theta=pi/2, W=I -> [[0,-1],[2,0]] in the
    paper's D_in x D_out layout; our [N,K] layout is its transpose."""
    ex = GOLD["bundle_2x2"]
    alpha = np.array(ex["alpha"])
    s = (1.0 / alpha).astype(np.float32)
    theta = np.array([[[ex["theta"]]]], dtype=np.float32)
    pairs = np.array([[[ex["pair"]]]], dtype=np.int16)
    W = np.eye(2, dtype=np.float16)                        # paper W = I -> W_pt = I^T = I
    V = O.fold(W, s, theta, pairs, g=2)
    expect = np.array(ex["TW_paper_layout"]).T
    np.testing.assert_allclose(V, expect, atol=2e-7)       # fp32 theta: cos(fl32(pi/2)) ~ -4.4e-8


@pytest.mark.parametrize("g,L", [(8, 3), (32, 8), (128, 8)])
def test_fold_matches_dense_givens_product(g, L):
    """Brute force: the oracle's vectorised fold equals the explicit product of dense
    Givens matrices in the paper's order G_L..G_1 diag(alpha) (Eq. 3, Eq. 8)."""
    K = g * 2
    p = synth.make_problem(8, K, seed=11, g=g, n_rot=L, n_pairs=g // 2)
    V = O.fold(p["W"], p["s"], p["theta"], p["pairs"], g=g)
    W = p["W"].astype(np.float64)
    for gam in range(2):
        M = dense_transform(1.0 / p["s"][gam * g:(gam + 1) * g].astype(np.float64),
                            p["theta"][gam], p["pairs"][gam])
        ref = W[:, gam * g:(gam + 1) * g] @ M.T        # each row w_n -> M w_n
        np.testing.assert_allclose(V[:, gam * g:(gam + 1) * g], ref, rtol=0, atol=1e-12)
        np.testing.assert_allclose(O.materialize(p["s"][gam * g:(gam + 1) * g], p["theta"][gam],
                                                 p["pairs"][gam]), M, atol=1e-13)


@pytest.mark.parametrize("g", [8, 32, 128])
def test_orthogonality_and_determinant(g):
    """alpha = 1: the transform is a product of rotations, M^T M = I, det M = +1
    (PAPER.md:87 'orthogonal matrix')."""
    p = synth.make_problem(1, g, seed=5, g=g, n_rot=8, n_pairs=g // 2, s_mode="ones")
    M = O.materialize(p["s"], p["theta"][0], p["pairs"][0])
    assert np.max(np.abs(M.T @ M - np.eye(g))) < 1e-13
    assert abs(np.linalg.det(M) - 1.0) < 1e-10


def test_norm_preservation_alpha_one():
    p = synth.make_problem(32, 512, seed=6, s_mode="ones")
    V = O.fold(p["W"], p["s"], p["theta"], p["pairs"])
    W = p["W"].astype(np.float64).reshape(32, 4, 128)
    np.testing.assert_allclose(np.linalg.norm(V.reshape(32, 4, 128), axis=2), np.linalg.norm(W, axis=2),
                               rtol=1e-13)


def test_pair_order_within_rotation_is_irrelevant_bitwise():
    """Pairs of one independent rotation commute (Def. 2, PAPER.md:143 'fully
    parallelizable'); permuting slot order gives a bitwise-equal result."""
    p = synth.make_problem(16, 256, seed=7)
    rng = np.random.default_rng(0)
    perm = rng.permutation(p["pairs"].shape[2])
    V1 = O.fold(p["W"], p["s"], p["theta"], p["pairs"])
    V2 = O.fold(p["W"], p["s"], p["theta"][:, :, perm], p["pairs"][:, :, perm])
    assert np.array_equal(V1, V2)


def test_rotation_order_matters():
    """Rotations of different layers do NOT commute (PAPER.md:141 'not commutative'):
    reversing the layer order changes the result (guards against a silently
    order-insensitive implementation)."""
    p = synth.make_problem(8, 128, seed=8)
    V1 = O.fold(p["W"], p["s"], p["theta"], p["pairs"])
    V2 = O.fold(p["W"], p["s"], p["theta"][:, ::-1], p["pairs"][:, ::-1])
    assert np.max(np.abs(V1 - V2)) > 1e-3


@pytest.mark.parametrize("seed", range(5))
def test_equivalent_transform_exactness(seed):
    """Eq. 2: (X T^-1)(T W) = X W before quantisation; the north_star's
    '(W T^-1)(T x) = W x exactly'.  fp64, relative 1e-12."""
    p = synth.make_problem(64, 512, B=7, seed=seed)
    V = O.fold(p["W"], p["s"], p["theta"], p["pairs"])
    U = O.transform_activations(p["x"], p["s"], p["theta"], p["pairs"])
    y_t = U @ V.T
    y = O.linear_fp(p["x"], p["W"])
    assert np.max(np.abs(y_t - y)) <= 1e-12 * np.max(np.abs(y))


def test_activation_side_is_not_spec_prose_order():
    """dividing by alpha AFTER the rotations (SPEC.md:265 prose) breaks
    Eq. 2; the oracle's scale-first order satisfies it.  Pins the scale position."""
    p = synth.make_problem(8, 128, B=3, seed=9)
    V = O.fold(p["W"], p["s"], p["theta"], p["pairs"])
    U_bad = O.transform_activations(p["x"], np.ones_like(p["s"]), p["theta"], p["pairs"]) * p["s"][None, :]
    y = O.linear_fp(p["x"], p["W"])
    assert np.max(np.abs(U_bad @ V.T - y)) > 1e-3 * np.max(np.abs(y))


@pytest.mark.parametrize("g", [2, 4, 8])
def test_tiny_group_all_matchings(g):
    """Brute force on tiny groups: every perfect matching of g channels (g=4: 3, g=8: 105)
    as the first rotation, L in {1,2,3}; fold == dense Givens product and Eq. 2 holds."""
    chans = list(range(g))

    def matchings(cs):
        if not cs:
            yield []
            return
        a = cs[0]
        for k in range(1, len(cs)):
            b = cs[k]
            rest = cs[1:k] + cs[k + 1:]
            for m in matchings(rest):
                yield [(a, b)] + m

    all_m = list(matchings(chans))
    assert len(all_m) == {2: 1, 4: 3, 8: 105}[g]
    rng = np.random.default_rng(g)
    for mi, m in enumerate(all_m[:40]):
        for L in (1, 2, 3):
            P = g // 2
            pairs = np.full((1, L, P, 2), -1, np.int16)
            pairs[0, 0] = np.array(m)
            for t in range(1, L):                        # later rotations: random disjoint sub-matchings
                mm = all_m[rng.integers(len(all_m))]
                h = max(1, len(mm) // 2)
                pairs[0, t, :h] = np.array(mm[:h])
            theta = rng.uniform(-3, 3, size=(1, L, P)).astype(np.float32)
            s = np.exp(rng.uniform(-.5, .5, size=g)).astype(np.float32)
            W = rng.normal(0, 1, size=(3, g)).astype(np.float16)
            x = rng.normal(0, 1, size=(2, g)).astype(np.float16)
            V = O.fold(W, s, theta, pairs, g=g)
            M = dense_transform(1.0 / s.astype(np.float64), theta[0], pairs[0])
            np.testing.assert_allclose(V, W.astype(np.float64) @ M.T, atol=1e-13)
            U = O.transform_activations(x, s, theta, pairs, g=g)
            np.testing.assert_allclose(U @ V.T, x.astype(np.float64) @ W.astype(np.float64).T, atol=1e-12)


# ------------------------------------------------------------------ RTN pins (Eq. 1)
def _group(vals, g=128):
    v = np.zeros((1, g))
    v[0, :len(vals)] = vals
    v[0, len(vals):] = vals[0]
    return v


def test_rtn_spec_range_example():
    ex = GOLD["rtn_range_example"]
    v = _group([ex["group_min"], ex["group_max"], 0.5])
    q, S, z = O.rtn_groups(v)
    assert float(S[0, 0]) == ex["S_fp16"]
    assert int(z[0, 0]) == ex["z"]
    t = GOLD["rtn_tie_example"]
    v2 = _group([ex["group_min"], ex["group_max"], t["v_fp16"]])
    q2, S2, z2 = O.rtn_groups(v2)
    assert int(q2[0, 2]) == t["code"]
    d = GOLD["rtn_dequant_example"]
    deq = O.dequantize(q2, S2, z2)
    assert abs(deq[0, 2] - d["value"]) < 1e-3                  # (7-5)*0.19995 = 0.3999
    assert abs(deq[0, 2] - t["v_fp16"]) <= float(S2[0, 0]) / 2 + 1e-12


def test_rtn_identity_grid():
    ex = GOLD["rtn_identity_grid"]
    vals = np.tile(np.arange(16.0), 8)
    q, S, z = O.rtn_groups(vals[None, :])
    assert float(S[0, 0]) == ex["S"] and int(z[0, 0]) == ex["z"]
    assert np.array_equal(q[0], vals.astype(np.uint8))


def test_rtn_all_zero_group():
    q, S, z = O.rtn_groups(np.zeros((2, 256)))
    assert np.all(q == 0) and np.all(z == 0) and np.all(S == np.float16(2 ** -24))


def test_rtn_zero_point_clamp_all_positive():
    """Q11: z = -round(min/S) clamped to [0, 15]; an all-positive group has
    unclamped z = -1.  Hand-computed S, z and codes (golden file)."""
    ex = GOLD["rtn_all_positive_group"]
    vals = np.array(ex["values"], dtype=np.float64)
    v = np.tile(vals, 8)[None, :]                                   # 128 values, 8 copies of 1..16
    q, S, z = O.rtn_groups(v)
    assert float(S[0, 0]) == ex["S"] and int(z[0, 0]) == ex["z"]
    assert np.array_equal(q[0, :16], np.array(ex["codes"], dtype=np.uint8))


def test_rtn_zero_point_clamp_all_negative():
    """Q11: an all-negative group has unclamped z = 16 -> 15, and the code clamp comes AFTER
    adding z (clamping round(v/S) first would give 15 everywhere)."""
    ex = GOLD["rtn_all_negative_group"]
    v = np.tile(np.array(ex["values"], dtype=np.float64), 8)[None, :]
    q, S, z = O.rtn_groups(v)
    assert float(S[0, 0]) == ex["S"] and int(z[0, 0]) == ex["z"]
    assert np.array_equal(q[0, :16], np.array(ex["codes"], dtype=np.uint8))
    deq = O.dequantize(q, S, z)
    # in-range values dequantise exactly; -16 is below the clamped grid [-15, 0]
    assert np.array_equal(deq[0, 1:16], np.array(ex["values"][1:], dtype=np.float64))
    assert deq[0, 0] == -15.0


@pytest.mark.parametrize("sign", ["pos", "neg"])
def test_rtn_constant_nonzero_group(sign):
    """Q10 (constant group -> s = eps, z clamped, all codes equal) with eps =
    2^-24 (the fp16 floor).  Hand-computed: c = 0.5 -> z = 0, codes 15; c = -0.5 -> z = 15,
    codes 0."""
    ex = GOLD["rtn_constant_group"]
    c = ex["c_" + sign]
    q, S, z = O.rtn_groups(np.full((3, 256), c))
    assert np.all(S.astype(np.float64) == ex["S"]) and ex["S"] == 2.0 ** -24
    assert np.all(z == ex[sign]["z"]) and np.all(q == ex[sign]["code"])


def test_fp16_single_rounding():
    """Q8: the stored scale is ONE round-to-nearest-even from fp64; via fp32 it would
    double-round (1 + 2^-11 + 2^-40 -> 1.0009765625 direct, 1.0 via fp32)."""
    v = 1.0 + 2.0 ** -11 + 2.0 ** -40
    assert float(np.float64(v).astype(np.float16)) == 1.0009765625
    assert float(np.float32(v).astype(np.float16)) == 1.0
    # through rtn_groups: a group whose s64 = v exactly
    grp = np.zeros((1, 128))
    grp[0, 1] = 15.0 * v
    _, S, _ = O.rtn_groups(grp)
    s64 = (15.0 * v - 0.0) / 15.0
    assert float(S[0, 0]) == float(np.float64(s64).astype(np.float16))


@pytest.mark.parametrize("bits", [2, 3, 4, 8])
def test_rtn_matches_scalar_bruteforce(bits):
    """SPEC.md:680 acceptance #3: Eq. 1 codes equal an exhaustive nearest-grid-point
    search for every in-range element; dequant error <= S/2; codes monotone."""
    rng = np.random.default_rng(bits)
    qmax = 2 ** bits - 1
    for trial in range(10):
        V = rng.normal(0, 1, size=(16, 128)) * rng.uniform(0.01, 5)
        q, S, z = O.rtn_groups(V, bits=bits)
        for n in range(16):
            Sn, zn = float(S[n, 0]), int(z[n, 0])
            grid = (np.arange(qmax + 1) - zn) * Sn
            lo, hi = grid[0], grid[-1]
            for k in range(128):
                v = V[n, k]
                if v < lo or v > hi:
                    continue
                d = np.abs(grid - v)
                best = int(np.argmin(d))
                srt = np.sort(d)
                if srt[1] - srt[0] < 1e-9 * Sn:             # tie: excluded
                    continue
                assert q[n, k] == best
                assert abs(grid[q[n, k]] - v) <= Sn / 2 + 1e-15
            order = np.argsort(V[n])
            assert np.all(np.diff(q[n, order].astype(int)) >= 0)


def test_rtn_matches_torch_fake_quantize():
    """Independent library routine: torch.fake_quantize_per_channel_affine with the
    oracle's (S, z) reproduces the oracle's dequantised values (fp32, ties excluded)."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(1)
    V = rng.normal(0, 0.02, size=(32, 512))
    q, S, z = O.rtn_groups(V)
    deq = O.dequantize(q, S, z)
    Vg = torch.from_numpy(V.reshape(-1, 128).astype(np.float32))
    sc = torch.from_numpy(S.reshape(-1).astype(np.float32))
    zp = torch.from_numpy(z.reshape(-1).astype(np.int32))
    fq = torch.fake_quantize_per_channel_affine(Vg, sc, zp, 0, 0, 15).numpy().reshape(32, 512)
    ratio = V.reshape(32, 4, 128) / S.astype(np.float64)[:, :, None]
    near_tie = (np.abs(ratio - np.floor(ratio) - 0.5) < 1e-5).reshape(32, 512)
    ok = ~near_tie
    np.testing.assert_allclose(fq[ok], deq[ok], rtol=0, atol=1e-7)


def test_pack_reduces_to_plain_rtn():
    """theta = 0, s = 1  =>  paro_pack == plain group-wise RTN of W, bit for bit
    (the north_star's reduction; PAPER.md:581 init)."""
    p = synth.make_problem(48, 384, seed=12, theta_mode="zero", s_mode="ones", zero_group=True)
    pk = O.oracle_pack(p["W"], p["s"], p["theta"], p["pairs"])
    q, S, z = O.rtn_groups(p["W"].astype(np.float64))
    assert np.array_equal(pk["codes"], q) and np.array_equal(pk["scales"], S) and np.array_equal(pk["zeros"], z)


def test_linear_scalar_loop_bruteforce():
    """oracle_linear's dequant-dot equals a pure-Python scalar loop of
    y[b,n] = sum_gamma S * sum_k (q - z) * x'[b,k] on a tiny case."""
    p = synth.make_problem(5, 256, B=2, seed=13, with_bias=True)
    pk = O.oracle_pack(p["W"], p["s"], p["theta"], p["pairs"])
    y = O.oracle_linear(p["x"], pk, p["s"], p["theta"], p["pairs"], bias=p["bias"])
    U = O.transform_activations(p["x"], p["s"], p["theta"], p["pairs"])
    for b in range(2):
        for n in range(5):
            acc = 0.0
            for gam in range(2):
                inner = 0.0
                for k in range(128):
                    inner += (int(pk["codes"][n, gam * 128 + k]) - int(pk["zeros"][n, gam])) * U[b, gam * 128 + k]
                acc += float(pk["scales"][n, gam]) * inner
            acc += float(p["bias"][n])
            assert abs(acc - y[b, n]) <= 1e-12 * max(1.0, abs(acc))


def test_quantised_output_close_to_fp_output():
    """Sanity (not a parity tolerance): W4 g128 output error vs the unquantised
    product is of the expected order (~10 %, SURVEY.md Q13 probe), and not larger
    than plain RTN's by much."""
    p = synth.make_problem(256, 1024, B=4, seed=14)
    pk = O.oracle_pack(p["W"], p["s"], p["theta"], p["pairs"])
    y = O.oracle_linear(p["x"], pk, p["s"], p["theta"], p["pairs"])
    yfp = O.linear_fp(p["x"], p["W"])
    e = O.normwise_error(y, yfp)
    assert 0.005 < e < 0.4


# ------------------------------------------------------------------ validation (SURVEY 8(b) errors)
def _bad(p, **kw):
    q = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in p.items()}
    q.update(kw)
    return q


@pytest.mark.parametrize("case,kind", [
    ("dup_channel", "pairs"), ("i_gt_j", "pairs"), ("half_pad", "pairs"), ("cross_layer_repeat", "pairs"),
    ("oob", "pairs"), ("s_nonpos", "invalid_argument"), ("s_nan", "invalid_argument"),
    ("theta_inf", "invalid_argument"), ("k_ragged", "unsupported"),
])
def test_validation_errors(case, kind):
    p = synth.make_problem(4, 256, seed=15)
    pr, th, s, W = p["pairs"].copy(), p["theta"].copy(), p["s"].copy(), p["W"]
    if case == "dup_channel":
        pr[0, 0, 1] = pr[0, 0, 0]
    elif case == "i_gt_j":
        pr[1, 2, 3] = pr[1, 2, 3][::-1]
    elif case == "half_pad":
        pr[0, 1, 5, 1] = -1
    elif case == "cross_layer_repeat":
        # put layer 0's first pair into layer 1, replacing a pair that uses the same channels
        a, b = pr[0, 0, 0]
        for t in range(pr.shape[2]):
            if a in pr[0, 1, t] or b in pr[0, 1, t]:
                pr[0, 1, t] = -1
        pr[0, 1, 0] = (a, b)
    elif case == "oob":
        pr[0, 0, 0, 1] = 128
    elif case == "s_nonpos":
        s[3] = 0.0
    elif case == "s_nan":
        s[3] = np.nan
    elif case == "theta_inf":
        th[0, 0, 0] = np.inf
    if case == "k_ragged":
        with pytest.raises(O.OracleError) as e:
            O.validate_transform(200, s[:200], th, pr)
    else:
        with pytest.raises(O.OracleError) as e:
            O.oracle_pack(W, s, th, pr)
    assert e.value.kind == kind


# ------------------------------------------------------------------ input generator structure
def test_alg_a1_structure():
    """SPEC.md:681 acceptance #4 / PAPER.md:216: at g=128, K=8, N=64 the first rotation has
    exactly 64 pairs; pairs disjoint within a rotation; no pair repeated; i<j."""
    pr = synth.select_pairs(6, seed=3)
    assert pr.shape == (6, 8, 64, 2)
    for gam in range(6):
        assert np.all(pr[gam, 0] >= 0)
        seen = set()
        for t in range(8):
            used = []
            for p in range(64):
                i, j = map(int, pr[gam, t, p])
                if i < 0:
                    assert j < 0
                    continue
                assert 0 <= i < j < 128
                used += [i, j]
                assert (i, j) not in seen
                seen.add((i, j))
            assert len(used) == len(set(used))
    assert np.array_equal(pr, synth.select_pairs(6, seed=3))


def test_param_ratio():
    """n/2 parameters per independent rotation = 1/(n-1) of a full rotation."""
    ex = GOLD["param_ratio"]
    n = ex["n"]
    assert abs((n / 2) / (n * (n - 1) / 2) - ex["ratio"]) < 1e-15
