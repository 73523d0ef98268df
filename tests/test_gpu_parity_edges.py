"""GPU parity, edge structure and the launch configurations the bench times (SURVEY.md 8(c)
P5/P7/P9 and VERDICT r1 "parity gaps"): one-signed and constant weight groups (Eq. 1's
zero-point clamp and scale floor, Q10/Q11), an all-zero activation group (the fixed-point
exponent floor of the IMMA decode path), activations near the fp16 range, on-the-fly
transforms with short rotations in every kernel family, full-size multi-linear launches
(70B gate+up, Qwen3-4B q/k/v at 16 tokens) and the NCCL all-gather path at world = 1.

Bar (north_star): codes / fp16 scales / zeros bit-exact; outputs within normwise 2e-3 of
the quantised fp64 oracle."""
import numpy as np
import pytest

import oracle as O
import synth

from test_gpu_parity import TOL, check_pack, dev_tensors, x_as_used

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def paro():
    import paper_2511_10645_b200 as m
    return m


def run_and_check(paro, p, t, packed, ref, flags=0, **kw):
    y = paro.paro_linear(t["x"], packed, bias=t["bias"], flags=flags, **kw)
    y_ref = O.oracle_linear(x_as_used(t), ref, p["s"], p["theta"], p["pairs"], bias=p["bias"])
    err = O.normwise_error(y.float().cpu().numpy(), y_ref)
    assert err <= TOL, f"normwise error {err:.3e}"
    return err


# decode B = 1 (fused K-split kernel), B = 2 (cluster-shared-transform kernel), B = 5 and 16
# (K-split kernel with the transform pre-kernel), B = 300 (prefill tcgen05 GEMM)
PATHS = [(1, 0), (2, 0), (5, 0), (16, 0), (300, "gemm")]


@pytest.mark.parametrize("B,path", PATHS)
def test_one_signed_and_constant_groups(paro, B, path):
    """All-positive, all-negative and constant-0.5 weight groups after the fold: z = 0 / 15
    (clamped), S = 2^-24 for the constant group; bit-exact pack, linear within tolerance."""
    p = synth.make_problem(256, 1024, B, seed=301, special_groups=True, with_bias=True)
    t = dev_tensors(p)
    packed, ref = check_pack(paro, p, t)
    assert np.all(ref["zeros"][:, 2] == 0) and np.all(ref["zeros"][:, 3] == 15)
    assert np.all(ref["scales"][:, 4].astype(np.float64) == 2.0 ** -24) and np.all(ref["codes"][:, 512:640] == 15)
    run_and_check(paro, p, t, packed, ref, paro.PARO_LINEAR_FORCE_GEMM if path == "gemm" else 0)


@pytest.mark.parametrize("B,path", PATHS)
def test_zero_activation_group(paro, B, path):
    """x = 0 on a whole group: max|x'| = 0 takes the exponent floor (E = -100) of the
    fixed-point digits; the group contributes exactly 0."""
    p = synth.make_problem(320, 1024, B, seed=302, x_zero_group=True)
    t = dev_tensors(p)
    packed, ref = check_pack(paro, p, t)
    run_and_check(paro, p, t, packed, ref, paro.PARO_LINEAR_FORCE_GEMM if path == "gemm" else 0)


@pytest.mark.parametrize("B,path", PATHS)
def test_activations_near_fp16_range(paro, B, path):
    """One channel per group at +-30000 (|s x| up to 49500 < 65504, paro.h precondition):
    the fp16 x' of the prefill / B = 2..4 paths and the per-group fixed point of the IMMA
    path keep their accuracy at the top of the range."""
    p = synth.make_problem(256, 1024, B, seed=303, x_big=30000.0)
    t = dev_tensors(p)
    packed, ref = check_pack(paro, p, t)
    run_and_check(paro, p, t, packed, ref, paro.PARO_LINEAR_FORCE_GEMM if path == "gemm" else 0)


@pytest.mark.parametrize("B,path", [(1, 0), (2, 0), (5, 0), (16, 0), (40, "gemm")])
def test_on_the_fly_short_rotations(paro, B, path):
    """On-the-fly transform (s / theta / pairs given to paro_linear) with 20 % absent slots:
    the prepared tables must keep every index in range (identity pairs on a channel the
    rotation leaves untouched) in every kernel family."""
    p = synth.force_short_layers(synth.make_problem(384, 1024, B, seed=304), seed=5, frac=0.2)
    t = dev_tensors(p)
    packed, ref = check_pack(paro, p, t)
    flags = (paro.PARO_LINEAR_FORCE_GEMM if path == "gemm" else 0) | paro.PARO_LINEAR_PDL
    run_and_check(paro, p, t, packed, ref, flags, s=t["s"], theta=t["theta"], pairs=t["pairs"])


def _multi_sampled(paro, shapes, B, seed, nrows=48, flags=0):
    """Full-size multi-linear launch (one x, one transform per linear); oracle on sampled rows."""
    K = shapes[0][1]
    probs = [synth.make_problem(N, K, B, seed=seed + i) for i, (N, _) in enumerate(shapes)]
    x = probs[0]["x"]
    xt = torch.from_numpy(x).cuda()
    packs, refs, rows_l = [], [], []
    for i, p in enumerate(probs):
        t = dev_tensors(p)
        rows = np.sort(np.random.default_rng(seed + i).choice(p["N"], size=nrows, replace=False))
        pk, ref = check_pack(paro, p, t, rows=rows)
        packs.append(pk)
        refs.append(ref)
        rows_l.append(rows)
        del t
    ys = paro.paro_linear_multi(xt, packs, flags=flags)
    torch.cuda.synchronize()
    for p, ref, rows, y in zip(probs, refs, rows_l, ys):
        y_ref = O.oracle_linear(x, ref, p["s"], p["theta"], p["pairs"])
        err = O.normwise_error(y.float().cpu().numpy()[:, rows], y_ref)
        assert err <= TOL, f"N={p['N']}: normwise error {err:.3e}"


def test_llama70b_gate_up_multi(paro):
    """configs[4] at one GPU as bench.py times it: gate+up (28672 x 8192 each) in ONE decode
    launch at bs = 1 -- clusters of 3840+ rows take the shared-atomic row-partial path."""
    _multi_sampled(paro, [(28672, 8192), (28672, 8192)], 1, 400, flags=paro.PARO_LINEAR_PDL)


@pytest.mark.parametrize("B", [16, 8])
def test_qwen3_4b_qkv_multi_b16(paro, B):
    """configs[2] at bs 16 / 8: Qwen3-4B q/k/v (4096 / 1024 / 1024 x 2560) in one launch."""
    _multi_sampled(paro, [(4096, 2560), (1024, 2560), (1024, 2560)], B, 410, flags=paro.PARO_LINEAR_PDL)


@pytest.mark.parametrize("B", [1, 3])
def test_allgather_world1(paro, B):
    """SURVEY.md 8(e) on the one-GPU box: paro_linear_allgather with a world = 1 NCCL
    communicator (ncclAllGather over one rank, then the rank-major permute for B > 1)."""
    p = synth.make_problem(512, 1024, B, seed=420 + B, with_bias=True)
    t = dev_tensors(p)
    packed, ref = check_pack(paro, p, t)
    uid = paro.paro_comm_unique_id()
    comm = paro.paro_comm_init(uid, 0, 1)
    try:
        y = paro.paro_linear_allgather(t["x"], packed, comm, 0, 1, bias_shard=t["bias"], flags=paro.PARO_LINEAR_PDL)
        torch.cuda.synchronize()
        paro.paro_comm_check(comm)
    finally:
        paro.paro_comm_destroy(comm)
    y_ref = O.oracle_linear(p["x"], ref, p["s"], p["theta"], p["pairs"], bias=p["bias"])
    assert O.normwise_error(y.float().cpu().numpy(), y_ref) <= TOL


@pytest.mark.parametrize("group", ["qkv", "o", "gate_up", "down"])
def test_llama8b_bench_step_launches(paro, group):
    """configs[1] exactly as bench.py's step launches it: the four paro_linear_multi launches
    of the LLaMA-3-8B decode layer at bs = 1 with PDL (q/k/v at K = 4096 in one launch, o,
    gate+up in one launch, down at K = 14336); oracle on sampled rows of every linear."""
    shapes = {"qkv": [(4096, 4096), (1024, 4096), (1024, 4096)], "o": [(4096, 4096)],
              "gate_up": [(14336, 4096), (14336, 4096)], "down": [(4096, 14336)]}[group]
    _multi_sampled(paro, shapes, 1, 500 + len(group), flags=paro.PARO_LINEAR_PDL)


def test_allgather_p2p_world1(paro):
    """SURVEY.md 8(f) NEXT #4 at world = 1: the NVLink-native exchange (the B = 1 GEMV epilogue
    storing into every rank's y_full through peer pointers, flags released by the last CTA, the
    wait kernel) with this process as the only rank; repeated calls advance the epoch."""
    p = synth.make_problem(512, 1024, 1, seed=430, with_bias=True)
    t = dev_tensors(p)
    packed, ref = check_pack(paro, p, t)
    buf = paro.p2p_buffer(512, 1, torch.float16)
    assert len(paro.paro_ipc_get_handle(buf)) == 64
    for _ in range(3):
        y = paro.paro_linear_allgather_p2p(t["x"], packed, [buf.data_ptr()], 0, 1, buf, bias_shard=t["bias"],
                                           flags=paro.PARO_LINEAR_PDL)
    torch.cuda.synchronize()
    y_ref = O.oracle_linear(p["x"], ref, p["s"], p["theta"], p["pairs"], bias=p["bias"])
    assert O.normwise_error(y.float().cpu().numpy(), y_ref) <= TOL
    words = buf[-256:].view(torch.int32).cpu().numpy()
    assert words[32 + 0] == 3 and words[0] == 3, "three exchanges: flag and epoch at 3"
