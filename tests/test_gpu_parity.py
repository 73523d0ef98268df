"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle on the same seeded
inputs.  Bar (north_star): packed codes / fp16 scales / zeros bit-exact; outputs within
normwise max-relative error 2e-3 of the quantised oracle."""
import math
import zlib

import numpy as np
import pytest

import oracle as O
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 2e-3


@pytest.fixture(scope="module")
def paro():
    import paper_2511_10645_b200 as m
    return m


def dev_tensors(p):
    d = torch.device("cuda")
    out = dict(W=torch.from_numpy(p["W"]).to(d), s=torch.from_numpy(p["s"]).to(d),
               theta=torch.from_numpy(p["theta"]).to(d), pairs=torch.from_numpy(p["pairs"]).to(d))
    if p["x"].dtype == np.float32:          # bf16 request
        out["x"] = torch.from_numpy(p["x"]).to(d).to(torch.bfloat16)
    else:
        out["x"] = torch.from_numpy(p["x"]).to(d)
    out["bias"] = None if p["bias"] is None else torch.from_numpy(p["bias"]).to(d)
    return out


def x_as_used(t):
    """The exact activation values the GPU saw (bf16 rounding happens in torch)."""
    return t["x"].float().cpu().numpy()


def check_pack(paro, p, t, rows=None):
    packed = paro.paro_pack(t["W"], t["s"], t["theta"], t["pairs"])
    codes, scales, zeros = (a.cpu().numpy() for a in paro.paro_unpack_logical(packed))
    Wn = p["W"] if rows is None else p["W"][rows]
    ref = O.oracle_pack(Wn, p["s"], p["theta"], p["pairs"])
    if rows is not None:
        codes, scales, zeros = codes[rows], scales[rows], zeros[rows]
    assert np.array_equal(scales.view(np.uint16), ref["scales"].view(np.uint16)), \
        f"{np.sum(scales.view(np.uint16) != ref['scales'].view(np.uint16))} scales differ"
    assert np.array_equal(zeros, ref["zeros"]), f"{np.sum(zeros != ref['zeros'])} zeros differ"
    assert np.array_equal(codes, ref["codes"]), f"{np.sum(codes != ref['codes'])} codes differ"
    return packed, ref


CASES = {
    "P1_c1": dict(N=256, K=256, B=1),
    "P2_identity": dict(N=256, K=256, B=1, theta_mode="zero", s_mode="ones"),
    "P4_quarter": dict(N=256, K=256, B=1, theta_mode="quarter"),
    "P4_eighth": dict(N=256, K=256, B=1, theta_mode="eighth"),
    "P5_outliers_zero_group": dict(N=1024, K=4096, B=3, zero_group=True),
    "ragged_rows": dict(N=389 * 2 + 1, K=640, B=2, with_bias=True),
    "qwen_k2560": dict(N=1024, K=2560, B=1),
    "bigK_9728": dict(N=512, K=9728, B=1),
}


@pytest.mark.parametrize("name", list(CASES))
def test_pack_and_linear(paro, name):
    kw = dict(CASES[name])
    N, K, B = kw.pop("N"), kw.pop("K"), kw.pop("B")
    p = synth.make_problem(N, K, B, seed=zlib.crc32(name.encode()) % 1000, **kw)
    t = dev_tensors(p)
    packed, ref = check_pack(paro, p, t)
    y = paro.paro_linear(t["x"], packed, bias=t["bias"])
    y_ref = O.oracle_linear(x_as_used(t), ref, p["s"], p["theta"], p["pairs"], bias=p["bias"])
    err = O.normwise_error(y.float().cpu().numpy(), y_ref)
    assert err <= TOL, f"{name}: normwise error {err:.3e}"


def test_single_pair_closed_form(paro):
    p = synth.single_pair_problem(N=256, K=256, group=1, layer=3, i=5, j=77, theta=math.pi / 4)
    t = dev_tensors(p)
    packed, ref = check_pack(paro, p, t)
    y = paro.paro_linear(t["x"], packed)
    y_ref = O.oracle_linear(p["x"], ref, p["s"], p["theta"], p["pairs"])
    assert O.normwise_error(y.float().cpu().numpy(), y_ref) <= TOL


def test_short_layers(paro):
    p = synth.force_short_layers(synth.make_problem(512, 1024, 2, seed=21), seed=3, frac=0.2)
    t = dev_tensors(p)
    packed, ref = check_pack(paro, p, t)
    y = paro.paro_linear(t["x"], packed)
    y_ref = O.oracle_linear(p["x"], ref, p["s"], p["theta"], p["pairs"])
    assert O.normwise_error(y.float().cpu().numpy(), y_ref) <= TOL


@pytest.mark.parametrize("n_rot", [0, 2, 4])
def test_fewer_rotations(paro, n_rot):
    """Table 6 varies #IR in {0, 2, 4, 8}."""
    p = synth.make_problem(256, 512, 1, seed=30 + n_rot, n_rot=max(n_rot, 1))
    if n_rot == 0:
        p["theta"] = p["theta"][:, :0]
        p["pairs"] = p["pairs"][:, :0]
    else:
        p["theta"] = p["theta"][:, :n_rot].copy()
        p["pairs"] = p["pairs"][:, :n_rot].copy()
    t = dev_tensors(p)
    packed, ref = check_pack(paro, p, t)
    y = paro.paro_linear(t["x"], packed)
    y_ref = O.oracle_linear(p["x"], ref, p["s"], p["theta"], p["pairs"])
    assert O.normwise_error(y.float().cpu().numpy(), y_ref) <= TOL


@pytest.mark.parametrize("B", [1, 2, 3, 4, 7, 16])
def test_batch_tails(paro, B):
    p = synth.make_problem(1024, 4096, B, seed=40 + B)
    t = dev_tensors(p)
    packed, ref = check_pack(paro, p, t)
    y = paro.paro_linear(t["x"], packed, flags=paro.PARO_LINEAR_FORCE_GEMV)
    y_ref = O.oracle_linear(p["x"], ref, p["s"], p["theta"], p["pairs"])
    assert O.normwise_error(y.float().cpu().numpy(), y_ref) <= TOL


@pytest.mark.parametrize("out_dtype", ["f16", "bf16", "f32"])
def test_dtypes(paro, out_dtype):
    """bf16 activations in, fp16/bf16/fp32 out.  bf16 output is compared against
    bf16_rne(y_ref) with 2e-3*max|y_ref| + half a bf16 ulp."""
    p = synth.make_problem(512, 1024, 2, seed=50, x_dtype="bf16")
    t = dev_tensors(p)
    packed, ref = check_pack(paro, p, t)
    odt = {"f16": torch.float16, "bf16": torch.bfloat16, "f32": torch.float32}[out_dtype]
    y = paro.paro_linear(t["x"], packed, out_dtype=odt).float().cpu().numpy()
    y_ref = O.oracle_linear(x_as_used(t), ref, p["s"], p["theta"], p["pairs"])
    if out_dtype == "bf16":
        yr = torch.from_numpy(y_ref).to(torch.bfloat16).float().numpy()
        ulp = np.abs(yr) * 2.0 ** -8
        assert np.all(np.abs(y - yr) <= TOL * np.max(np.abs(y_ref)) + ulp)
    else:
        assert O.normwise_error(y, y_ref) <= TOL


def test_no_rotation_flag_is_plain_w4a16(paro):
    """PARO_LINEAR_NO_ROTATION: u = x (overhead baseline) == oracle dot without the transform."""
    p = synth.make_problem(512, 1024, 1, seed=60)
    t = dev_tensors(p)
    packed, ref = check_pack(paro, p, t)
    y = paro.paro_linear(t["x"], packed, flags=paro.PARO_LINEAR_NO_ROTATION)
    y_ref = O.oracle_linear(p["x"], ref, p["s"], p["theta"], p["pairs"], rotate=False)
    assert O.normwise_error(y.float().cpu().numpy(), y_ref) <= TOL


def test_on_the_fly_transform(paro):
    p = synth.make_problem(256, 512, 2, seed=61)
    t = dev_tensors(p)
    packed, ref = check_pack(paro, p, t)
    y = paro.paro_linear(t["x"], packed, s=t["s"], theta=t["theta"], pairs=t["pairs"])
    y_ref = O.oracle_linear(p["x"], ref, p["s"], p["theta"], p["pairs"])
    assert O.normwise_error(y.float().cpu().numpy(), y_ref) <= TOL


def test_transform_activations(paro):
    """Activation side alone (Eq. 5 in column form): fp16 x' within fp16 rounding of the oracle."""
    p = synth.make_problem(8, 1024, 37, seed=62)
    t = dev_tensors(p)
    packed, _ = check_pack(paro, p, t)
    xp = paro.paro_transform_activations(t["x"], packed).float().cpu().numpy()
    ref = O.transform_activations(p["x"], p["s"], p["theta"], p["pairs"])
    assert np.all(np.abs(xp - ref) <= 2.0 ** -10 * np.abs(ref) + 1e-6 * np.max(np.abs(ref)))


@pytest.mark.parametrize("B,K", [(300, 1024), (37, 512), (129, 2048), (2048, 4096)])
def test_transform_activations_dense(paro, B, K):
    """Dense per-group form of the transform (M_g = R_L..R_1 diag(s_g) rounded to fp16, fp32
    accumulation): per channel within 2^-10 (|x'| + ||s . x_g||_2) of the oracle -- the fp16
    rounding of M (2^-11 relative per entry; rows of R have unit norm) plus the fp16 output.
    Ragged token tiles (B not a multiple of 128); bf16 x is refused (the dense form reads fp16)."""
    import torch
    p = synth.make_problem(8, K, B, seed=64 + B)
    t = dev_tensors(p)
    packed, _ = check_pack(paro, p, t)
    x = t["x"]
    with pytest.raises(paro.ParoError):
        paro.paro_transform_activations_dense(x.to(torch.bfloat16), packed)
    xin = x.float().cpu().numpy().astype(np.float64)
    xp = paro.paro_transform_activations_dense(x, packed).float().cpu().numpy()
    ref = O.transform_activations(xin, p["s"], p["theta"], p["pairs"])
    u = (xin * p["s"][None, :]).reshape(B, K // 128, 128)
    gnorm = np.repeat(np.sqrt((u ** 2).sum(-1)), 128, axis=1)
    assert np.all(np.abs(xp - ref) <= 2.0 ** -10 * (np.abs(ref) + gnorm))


def test_pack_errors(paro):
    p = synth.make_problem(64, 256, 1, seed=63)
    t = dev_tensors(p)
    bad = t["pairs"].clone()
    bad[0, 0, 1] = bad[0, 0, 0]
    with pytest.raises(paro.ParoError) as e:
        paro.paro_pack(t["W"], t["s"], t["theta"], bad)
    assert e.value.kind == "pairs"
    s_bad = t["s"].clone()
    s_bad[5] = -1.0
    with pytest.raises(paro.ParoError) as e:
        paro.paro_pack(t["W"], s_bad, t["theta"], t["pairs"])
    assert e.value.kind == "invalid_argument"
    W_bad = t["W"].clone()
    W_bad[3, 7] = float("inf")
    with pytest.raises(paro.ParoError) as e:
        paro.paro_pack(W_bad, t["s"], t["theta"], t["pairs"])
    assert e.value.kind == "invalid_argument"


@pytest.mark.parametrize("name,N,K", [("q_proj", 4096, 4096), ("down_proj", 4096, 14336), ("gate_proj", 14336, 4096),
                                      ("llama70b_gate", 28672, 8192), ("llama70b_down", 8192, 28672)])
def test_full_size_sampled(paro, name, N, K):
    """BASELINE configs[1] at full size, in the launch configuration bench.py times:
    pack bit-exact and outputs within tolerance on sampled rows (rows are independent
    in the fold, the RTN and the dot, so the oracle runs on the sampled rows only)."""
    p = synth.make_problem(N, K, 1, seed=70)
    t = dev_tensors(p)
    rows = np.sort(np.random.default_rng(0).choice(N, size=64, replace=False))
    packed, ref = check_pack(paro, p, t, rows=rows)
    # one workspace (garbage-filled) reused across calls, as a serving loop does (llama70b_down takes
    # the cross-cluster K split: its arrival counters, after s in packed.svec, must be back at zero
    # after every call)
    ws = torch.full((max(1, paro.paro_linear_workspace(1, N, K)),), 0xA5, dtype=torch.uint8, device="cuda")
    ys = [paro.paro_linear(t["x"], packed, flags=paro.PARO_LINEAR_PDL, workspace=ws) for _ in range(3)]
    y = ys[0].float().cpu().numpy()[:, rows]
    y_ref = O.oracle_linear(p["x"], ref, p["s"], p["theta"], p["pairs"])
    assert O.normwise_error(y, y_ref) <= TOL
    assert all(bool((ys[0] == yk).all()) for yk in ys[1:]), "repeated calls differ"
    assert int(packed.svec[K * 4:].count_nonzero()) == 0, "K-split counters not reset"


@pytest.mark.parametrize("B,N,K", [(300, 256, 512), (17, 384, 1024), (520, 1024, 4096)])
def test_prefill_gemm(paro, B, N, K):
    """Prefill path (B > 16): transform pre-stage + tcgen05 GEMM with TMEM dequant producer.  These
    shapes have few 256-token tiles, so each tile runs as two split-K halves on a cluster pair that
    exchange fp32 partials through DSMEM (fixed summation order): two calls are bit-identical."""
    p = synth.make_problem(N, K, B, seed=80 + B, with_bias=True)
    t = dev_tensors(p)
    packed, ref = check_pack(paro, p, t)
    y_ref = O.oracle_linear(p["x"], ref, p["s"], p["theta"], p["pairs"], bias=p["bias"])
    ys = [paro.paro_linear(t["x"], packed, bias=t["bias"], flags=paro.PARO_LINEAR_FORCE_GEMM) for _ in range(2)]
    err = O.normwise_error(ys[0].float().cpu().numpy(), y_ref)
    assert err <= TOL, f"prefill normwise error {err:.3e}"
    assert bool((ys[0] == ys[1]).all()), "split-K reduction is not deterministic"


@pytest.mark.parametrize("B,N", [(2048, 2560), (1500, 4096)])
def test_prefill_ragged_token_tiles(paro, B, N):
    """Prefill with a ragged last 256-token tile (2048 tokens over 20 row tiles; 1500 = 5 x 256 + 220)
    and a row-tile count that leaves the last tile round partly idle: every output against the
    oracle, fp16 and fp32 outputs."""
    K = 512
    p = synth.make_problem(N, K, B, seed=160 + B, with_bias=True)
    t = dev_tensors(p)
    packed, ref = check_pack(paro, p, t)
    y = paro.paro_linear(t["x"], packed, bias=t["bias"], flags=paro.PARO_LINEAR_FORCE_GEMM)
    y_ref = O.oracle_linear(p["x"], ref, p["s"], p["theta"], p["pairs"], bias=p["bias"])
    assert O.normwise_error(y.float().cpu().numpy(), y_ref) <= TOL
    yf = paro.paro_linear(t["x"], packed, bias=t["bias"], out_dtype=torch.float32, flags=paro.PARO_LINEAR_FORCE_GEMM)
    assert O.normwise_error(yf.cpu().numpy(), y_ref) <= TOL


@pytest.mark.parametrize("n_rot", [0, 2, 4])
def test_prefill_fewer_rotations(paro, n_rot):
    """Table 6 #IR in {0, 2, 4} on the prefill path: the dense transform's
    per-group matrix M_g = P R_L..R_1 diag(s_g) is built with L < 8 layers (L = 0: M_g = diag(s_g))."""
    B, N, K = 192, 512, 1024
    p = synth.make_problem(N, K, B, seed=130 + n_rot, n_rot=max(n_rot, 1))
    p["theta"] = p["theta"][:, :n_rot].copy()
    p["pairs"] = p["pairs"][:, :n_rot].copy()
    t = dev_tensors(p)
    packed, ref = check_pack(paro, p, t)
    y = paro.paro_linear(t["x"], packed, flags=paro.PARO_LINEAR_FORCE_GEMM)
    y_ref = O.oracle_linear(p["x"], ref, p["s"], p["theta"], p["pairs"])
    assert O.normwise_error(y.float().cpu().numpy(), y_ref) <= TOL


@pytest.mark.parametrize("out_dtype", ["bf16", "f32"])
def test_prefill_bf16_activations(paro, out_dtype):
    """bf16 x on the prefill path (the Givens transform pre-stage, not the fp16-only dense form),
    with bf16 / fp32 output; tolerance as test_dtypes."""
    p = synth.make_problem(768, 2048, 160, seed=140, x_dtype="bf16", with_bias=True)
    t = dev_tensors(p)
    packed, ref = check_pack(paro, p, t)
    odt = {"bf16": torch.bfloat16, "f32": torch.float32}[out_dtype]
    y = paro.paro_linear(t["x"], packed, bias=t["bias"], out_dtype=odt,
                         flags=paro.PARO_LINEAR_FORCE_GEMM).float().cpu().numpy()
    y_ref = O.oracle_linear(x_as_used(t), ref, p["s"], p["theta"], p["pairs"], bias=p["bias"])
    if out_dtype == "bf16":
        yr = torch.from_numpy(y_ref).to(torch.bfloat16).float().numpy()
        ulp = np.abs(yr) * 2.0 ** -8
        assert np.all(np.abs(y - yr) <= TOL * np.max(np.abs(y_ref)) + ulp)
    else:
        assert O.normwise_error(y, y_ref) <= TOL


@pytest.mark.parametrize("out_dtype", ["bf16", "f32"])
def test_k_split_bias_and_dtypes(paro, out_dtype):
    """The cross-cluster K split (one token, LLaMA-3-70B down_proj: 7 K slices on clusters of 2)
    with a bias and bf16 / fp32 output -- the last-arriver epilogue's other store paths -- on
    sampled rows; PDL launches alternating with an unsplit launch on the same garbage-filled
    workspace; the counters are back at zero afterwards."""
    N, K = 8192, 28672
    assert paro.paro_linear_workspace(1, N, K) == 7 * N * 4
    p = synth.make_problem(N, K, 1, seed=171, with_bias=True)
    t = dev_tensors(p)
    rows = np.sort(np.random.default_rng(3).choice(N, size=48, replace=False))
    packed, ref = check_pack(paro, p, t, rows=rows)
    p2 = synth.make_problem(1024, K, 1, seed=172)
    t2 = dev_tensors(p2)
    packed2 = paro.paro_pack(t2["W"], t2["s"], t2["theta"], t2["pairs"])
    odt = {"bf16": torch.bfloat16, "f32": torch.float32}[out_dtype]
    ws = torch.full((paro.paro_linear_workspace(1, N, K),), 0x5A, dtype=torch.uint8, device="cuda")
    ys = []
    for _ in range(2):
        ys.append(paro.paro_linear(t["x"], packed, bias=t["bias"], out_dtype=odt, flags=paro.PARO_LINEAR_PDL,
                                   workspace=ws))
        paro.paro_linear(t2["x"], packed2, flags=paro.PARO_LINEAR_PDL, workspace=ws)
    y = ys[0].float().cpu().numpy()[:, rows]
    y_ref = O.oracle_linear(p["x"], ref, p["s"], p["theta"], p["pairs"], bias=p["bias"][rows])
    if out_dtype == "bf16":
        yr = torch.from_numpy(y_ref).to(torch.bfloat16).float().numpy()
        assert np.all(np.abs(y - yr) <= TOL * np.max(np.abs(y_ref)) + np.abs(yr) * 2.0 ** -8)
    else:
        assert O.normwise_error(y, y_ref) <= TOL
    assert bool((ys[0] == ys[1]).all())
    assert int(packed.svec[K * 4:].count_nonzero()) == 0


@pytest.mark.parametrize("N,K", [(1000, 8192), (520, 16384), (96, 28672)])
def test_long_k_b1_all_rows(paro, N, K):
    """One token at long K (the shapes planned with clusters of 8 or with the K range split over
    several clusters): every row against the oracle, ragged row blocks, and two calls bit-identical
    (fixed-order reductions)."""
    p = synth.make_problem(N, K, 1, seed=150 + N)
    t = dev_tensors(p)
    packed, ref = check_pack(paro, p, t)
    ys = [paro.paro_linear(t["x"], packed, flags=paro.PARO_LINEAR_PDL) for _ in range(2)]
    y_ref = O.oracle_linear(p["x"], ref, p["s"], p["theta"], p["pairs"])
    assert O.normwise_error(ys[0].float().cpu().numpy(), y_ref) <= TOL
    assert bool((ys[0] == ys[1]).all())


@pytest.mark.parametrize("N,K", [(4096, 4096), (1024, 4096), (14336, 4096), (4096, 14336)])
def test_prefill_full_size_sampled(paro, N, K):
    """configs[3]: LLaMA-3-8B prefill 2048 tokens at the bench's shapes -- q/o (256 tiles), k/v
    (split-K cluster pairs), gate/up (896 tiles), down (dense transform over 112 groups) -- sampled
    tokens and rows against the oracle."""
    B = 2048
    p = synth.make_problem(N, K, B, seed=90)
    t = dev_tensors(p)
    rows = np.sort(np.random.default_rng(1).choice(N, size=32, replace=False))
    packed, ref = check_pack(paro, p, t, rows=rows)
    y = paro.paro_linear(t["x"], packed).float().cpu().numpy()
    toks = np.sort(np.random.default_rng(2).choice(B, size=64, replace=False))
    y_ref = O.oracle_linear(p["x"][toks], ref, p["s"], p["theta"], p["pairs"])
    assert O.normwise_error(y[toks][:, rows], y_ref) <= TOL


@pytest.mark.parametrize("B,N,K", [(8, 256, 14336), (16, 512, 9728), (5, 384, 2560), (12, 640, 4096), (2, 256, 28672)])
def test_k_split_tokens(paro, B, N, K):
    """Token counts routed to the K-split decode kernel (gemv1.cu) beyond one token, at the
    large-K shapes (clusters of 8): B = 5..16 in one launch, column sets of four tokens."""
    p = synth.make_problem(N, K, B, seed=80 + B)
    t = dev_tensors(p)
    packed, ref = check_pack(paro, p, t)
    y = paro.paro_linear(t["x"], packed, flags=paro.PARO_LINEAR_FORCE_GEMV)
    y_ref = O.oracle_linear(p["x"], ref, p["s"], p["theta"], p["pairs"])
    assert O.normwise_error(y.float().cpu().numpy(), y_ref) <= TOL


@pytest.mark.parametrize("N,K,B", [(96, 128, 1), (96, 128, 5), (200, 384, 1), (200, 384, 3), (4128, 640, 1)])
def test_k_split_edge_shapes(paro, N, K, B):
    """Edge shapes of the K-split decode kernel: one group (clusters of 1), an odd group count
    split unevenly over a cluster (G = 3, 5), ragged row blocks (N % 32 != 0), many row blocks
    over few groups."""
    p = synth.make_problem(N, K, B, seed=90 + N + B)
    t = dev_tensors(p)
    packed, ref = check_pack(paro, p, t)
    y = paro.paro_linear(t["x"], packed, flags=paro.PARO_LINEAR_FORCE_GEMV)
    y_ref = O.oracle_linear(p["x"], ref, p["s"], p["theta"], p["pairs"])
    assert O.normwise_error(y.float().cpu().numpy(), y_ref) <= TOL


@pytest.mark.parametrize("B", [1, 3, 6])
def test_linear_multi_shared_x(paro, B):
    """q/k/v-style: three linears with their own transforms reading the same x, one launch."""
    K = 1024
    shapes = [(512, K), (128, K), (256, K)]
    probs = [synth.make_problem(N, K, B, seed=100 + i, with_bias=(i == 1)) for i, (N, _) in enumerate(shapes)]
    x = probs[0]["x"]
    packs, refs = [], []
    for p in probs:
        t = dev_tensors(p)
        pk, ref = check_pack(paro, p, t)
        packs.append(pk)
        refs.append(ref)
    xt = torch.from_numpy(x).cuda()
    bias = [None if p["bias"] is None else torch.from_numpy(p["bias"]).cuda() for p in probs]
    ys = paro.paro_linear_multi(xt, packs, bias=bias)
    for p, ref, y in zip(probs, refs, ys):
        y_ref = O.oracle_linear(x, ref, p["s"], p["theta"], p["pairs"], bias=p["bias"])
        assert O.normwise_error(y.float().cpu().numpy(), y_ref) <= TOL


def test_copy_host_device(paro):
    """paro_copy (SM-driven copy for the serving loop): pinned host -> device -> pinned host and
    device -> device, byte-exact; PDL-chained with a decode launch in between; size errors."""
    import torch
    dev = torch.device("cuda")
    src = torch.randint(-30000, 30000, (3 * 4096 + 8,), dtype=torch.int16).pin_memory()
    d = torch.empty(src.shape, dtype=torch.int16, device=dev)
    d2 = torch.empty_like(d)
    back = torch.empty(src.shape, dtype=torch.int16).pin_memory()
    p = synth.make_problem(256, 1024, 1, seed=5)
    t = dev_tensors(p)
    packed, _ = check_pack(paro, p, t)
    paro.paro_copy(d, src, flags=paro.PARO_LINEAR_PDL)
    y = paro.paro_linear(t["x"], packed, flags=paro.PARO_LINEAR_PDL)
    paro.paro_copy(d2, d, flags=paro.PARO_LINEAR_PDL)
    paro.paro_copy(back, d2, flags=paro.PARO_LINEAR_PDL)
    torch.cuda.synchronize()
    assert torch.equal(back, src)
    assert torch.isfinite(y.float()).all()
    with pytest.raises(ValueError):
        paro.paro_copy(back[:-8], d2)
    with pytest.raises(paro.ParoError):
        paro.paro_copy(back[:-1], d2[:-1])  # 2 * 12295 bytes: not a multiple of 16
