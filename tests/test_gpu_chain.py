"""GPU parity of the persistent decode chain (paro_linear_chain, include/paro.h): stages run in
one launch with a grid-wide barrier between them, so a later stage may read an earlier stage's
y as its x.  Each stage is checked against the fp64 oracle applied to the EXACT activation the
GPU used (for a dependent stage: the previous stage's GPU output), so a barrier that let a stage
read a partial or stale y fails here.  Bar: normwise 2e-3."""
import numpy as np
import pytest

import oracle as O
import synth

from test_gpu_parity import TOL, check_pack, dev_tensors

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def paro():
    import paper_2511_10645_b200 as m
    return m


def _lin(paro, N, K, B, seed, nrows=None, bias=False, unit_gain=False):
    """A packed linear + its oracle pack (all rows, or `nrows` sampled rows).  unit_gain: W ~
    N(0, 1/K) without outlier channels, so repeated application keeps |y| ~ |x|."""
    p = synth.make_problem(N, K, B, seed=seed, with_bias=bias, outliers=not unit_gain)
    if unit_gain:
        p["W"] = (p["W"].astype(np.float64) * (1.0 / np.sqrt(K)) / 0.02).astype(np.float16)
    t = dev_tensors(p)
    rows = None if nrows is None or nrows >= N else \
        np.sort(np.random.default_rng(seed).choice(N, size=nrows, replace=False))
    pk, ref = check_pack(paro, p, t, rows=rows)
    return dict(p=p, packed=pk, ref=ref, rows=rows, bias=t["bias"])


def _check(lin, x_np, y):
    p, rows = lin["p"], lin["rows"]
    bias = None if p["bias"] is None else (p["bias"] if rows is None else p["bias"][rows])
    y_ref = O.oracle_linear(x_np, lin["ref"], p["s"], p["theta"], p["pairs"], bias=bias)
    yv = y.float().cpu().numpy()
    if rows is not None:
        yv = yv[:, rows]
    err = O.normwise_error(yv, y_ref)
    assert err <= TOL, f"N={p['N']} K={p['K']}: normwise error {err:.3e}"
    return err


@pytest.mark.parametrize("B", [1, 3, 8, 16])
def test_chain_dependent_stages(paro, B):
    """x -> [A: 1024 x 512] -> y0 -> [B1: 640 x 1024, B2: 256 x 1024] -> y1 -> [C: 384 x 640]:
    stage 1 reads stage 0's y, stage 2 reads stage 1's first output (B > 1: the later stages'
    transforms run inside the launch)."""
    A = _lin(paro, 1024, 512, B, 700, bias=True)
    B1 = _lin(paro, 640, 1024, B, 701)
    B2 = _lin(paro, 256, 1024, B, 702, bias=True)
    C = _lin(paro, 384, 640, B, 703)
    x = torch.from_numpy(A["p"]["x"]).cuda()
    y0 = torch.empty((B, 1024), dtype=torch.float16, device="cuda")
    y1 = torch.empty((B, 640), dtype=torch.float16, device="cuda")
    y2 = torch.empty((B, 256), dtype=torch.float16, device="cuda")
    y3 = torch.empty((B, 384), dtype=torch.float16, device="cuda")
    st = [paro.ChainStage(x, [A["packed"]], [y0], bias=[A["bias"]]),
          paro.ChainStage(y0, [B1["packed"], B2["packed"]], [y1, y2], bias=[None, B2["bias"]]),
          paro.ChainStage(y1, [C["packed"]], [y3])]
    paro.paro_linear_chain(st, flags=paro.PARO_LINEAR_PDL)
    torch.cuda.synchronize()
    _check(A, A["p"]["x"], y0)
    y0n = y0.float().cpu().numpy()
    _check(B1, y0n, y1)
    _check(B2, y0n, y2)
    _check(C, y1.float().cpu().numpy(), y3)


def test_chain_llama8b_layer(paro):
    """configs[1] as one chain: q/k/v (one stage), o, gate+up, down, with down reading up's
    output (a real dependency at full size); sampled rows against the oracle."""
    K = 4096
    q, k, v = (_lin(paro, N, K, 1, 710 + i, nrows=48) for i, N in enumerate((4096, 1024, 1024)))
    o = _lin(paro, 4096, 4096, 1, 713, nrows=48)
    gate, up = (_lin(paro, 14336, K, 1, 714 + i, nrows=48) for i in range(2))
    down = _lin(paro, 4096, 14336, 1, 716, nrows=48)
    x = torch.from_numpy(q["p"]["x"]).cuda()
    xo = torch.from_numpy(o["p"]["x"]).cuda()
    ys = {n: torch.empty((1, N), dtype=torch.float16, device="cuda")
          for n, N in (("q", 4096), ("k", 1024), ("v", 1024), ("o", 4096), ("g", 14336), ("u", 14336), ("d", 4096))}
    st = [paro.ChainStage(x, [q["packed"], k["packed"], v["packed"]], [ys["q"], ys["k"], ys["v"]]),
          paro.ChainStage(xo, [o["packed"]], [ys["o"]]),
          paro.ChainStage(x, [gate["packed"], up["packed"]], [ys["g"], ys["u"]]),
          paro.ChainStage(ys["u"], [down["packed"]], [ys["d"]])]
    ws = paro.chain_workspace(1, st)
    for _ in range(2):  # the barrier epoch advances per launch: a second call on the workspace works the same
        paro.paro_linear_chain(st, flags=paro.PARO_LINEAR_PDL, workspace=ws)
    torch.cuda.synchronize()
    xn = q["p"]["x"]
    for lin, name in ((q, "q"), (k, "k"), (v, "v"), (gate, "g"), (up, "u")):
        _check(lin, xn, ys[name])
    _check(o, o["p"]["x"], ys["o"])
    _check(down, ys["u"].float().cpu().numpy(), ys["d"])
    assert int(ws[:4].view(torch.int32)[0].item()) == 2, "one barrier epoch per persistent launch"


@pytest.mark.parametrize("B", [1, 5])
def test_chain_longer_than_one_launch(paro, B):
    """18 dependent stages (16 per persistent launch + a second launch): a ping-pong of two
    square linears, each stage reading the previous stage's y."""
    K = 256
    lins = [_lin(paro, K, K, B, 730 + i, unit_gain=True) for i in range(2)]
    x = torch.from_numpy(lins[0]["p"]["x"]).cuda()
    ys = [torch.empty((B, K), dtype=torch.float16, device="cuda") for _ in range(18)]
    st, prev = [], x
    for s in range(18):
        st.append(paro.ChainStage(prev, [lins[s % 2]["packed"]], [ys[s]]))
        prev = ys[s]
    paro.paro_linear_chain(st)
    torch.cuda.synchronize()
    prev_np = lins[0]["p"]["x"]
    for s in range(18):
        _check(lins[s % 2], prev_np, ys[s])
        prev_np = ys[s].float().cpu().numpy()


def test_chain_idle_ctas_and_ragged(paro):
    """A stage far smaller than the grid (2 row blocks: most CTAs idle), odd N, a wide stage,
    then an odd-group K (31 groups) -- different K per stage in one launch."""
    small = _lin(paro, 50, 256, 1, 740, bias=True)
    wide = _lin(paro, 4000, 256, 1, 741)
    tail = _lin(paro, 33, 3968, 1, 742)
    x = torch.from_numpy(small["p"]["x"]).cuda()
    xt = torch.from_numpy(tail["p"]["x"]).cuda()
    y0 = torch.empty((1, 50), dtype=torch.float16, device="cuda")
    y1 = torch.empty((1, 4000), dtype=torch.float16, device="cuda")
    y2 = torch.empty((1, 33), dtype=torch.float16, device="cuda")
    st = [paro.ChainStage(x, [small["packed"]], [y0], bias=[small["bias"]]),
          paro.ChainStage(x, [wide["packed"]], [y1]),
          paro.ChainStage(xt, [tail["packed"]], [y2])]
    paro.paro_linear_chain(st)
    torch.cuda.synchronize()
    _check(small, small["p"]["x"], y0)
    _check(wide, small["p"]["x"], y1)
    _check(tail, tail["p"]["x"], y2)


def test_chain_matches_separate_launches(paro):
    """A chain's outputs equal the same linears run as separate paro_linear_multi launches up
    to fp32 summation order (different cluster plans): within one fp16 ulp."""
    K = 2048
    a = _lin(paro, 2048, K, 1, 750, nrows=8)
    b = _lin(paro, 512, K, 1, 751, nrows=8)
    x = torch.from_numpy(a["p"]["x"]).cuda()
    y0 = torch.empty((1, 2048), dtype=torch.float16, device="cuda")
    y1 = torch.empty((1, 512), dtype=torch.float16, device="cuda")
    paro.paro_linear_chain([paro.ChainStage(x, [a["packed"]], [y0]), paro.ChainStage(y0, [b["packed"]], [y1])])
    r0 = paro.paro_linear_multi(x, [a["packed"]])[0]
    r1 = paro.paro_linear_multi(r0, [b["packed"]])[0]
    torch.cuda.synchronize()
    for u, v in ((y0, r0), (y1, r1)):
        assert O.normwise_error(u.float().cpu().numpy(), v.float().cpu().numpy().astype(np.float64)) <= 1e-3


def test_chain_errors(paro):
    a = _lin(paro, 256, 256, 1, 760)
    x = torch.zeros((17, 256), dtype=torch.float16, device="cuda")
    y = torch.empty((17, 256), dtype=torch.float16, device="cuda")
    with pytest.raises(paro.ParoError) as e:
        paro.paro_linear_chain([paro.ChainStage(x, [a["packed"]], [y])])
    assert e.value.kind == "unsupported"
    x1, y1 = x[:1], y[:1]
    with pytest.raises(paro.ParoError) as e:
        paro.paro_linear_chain([paro.ChainStage(x1, [a["packed"]], [y1])],
                               workspace=torch.zeros(16, dtype=torch.uint8, device="cuda"))
    assert e.value.kind == "invalid_argument"


@pytest.mark.parametrize("B", [2, 3, 5, 8, 12, 16])
def test_tcgen05_engine_single_and_chain(paro, B):
    """PARO_LINEAR_TCGEN05: the B > 1 tiles on tcgen05.mma kind::i8 (u8 codes in TMEM x s8 digits)
    -- one launch (stage-0 transform pre-kernel) and a dependent chain (in-kernel transform)."""
    A = _lin(paro, 1024, 2560, B, 770, bias=True)
    C = _lin(paro, 640, 1024, B, 771)
    x = torch.from_numpy(A["p"]["x"]).cuda()
    y = paro.paro_linear(x, A["packed"], bias=A["bias"], flags=paro.PARO_LINEAR_TCGEN05)
    torch.cuda.synchronize()
    _check(A, A["p"]["x"], y)
    y0 = torch.empty((B, 1024), dtype=torch.float16, device="cuda")
    y1 = torch.empty((B, 640), dtype=torch.float16, device="cuda")
    paro.paro_linear_chain([paro.ChainStage(x, [A["packed"]], [y0], bias=[A["bias"]]),
                            paro.ChainStage(y0, [C["packed"]], [y1])], flags=paro.PARO_LINEAR_TCGEN05)
    torch.cuda.synchronize()
    _check(A, A["p"]["x"], y0)
    _check(C, y0.float().cpu().numpy(), y1)
