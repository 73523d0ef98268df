"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): C1, q_proj-shaped decode at B in {1, 3, 16}, a multi-linear launch,
the on-the-fly transform, prefill at B = 300, and the pack.  Checks results against the
oracle too (so a sanitizer-perturbed run that computes garbage fails loudly).
Usage: compute-sanitizer --tool memcheck python tools/sanitize_cases.py [--quick]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2511_10645_b200 as paro  # noqa: E402
import synth  # noqa: E402


def dev(p):
    d = torch.device("cuda")
    return {k: torch.from_numpy(p[k]).to(d) for k in ("W", "s", "theta", "pairs", "x")}


def case(N, K, B, flags=0, seed=0, otf=False):
    p = synth.make_problem(N, K, B, seed=seed)
    t = dev(p)
    pk = paro.paro_pack(t["W"], t["s"], t["theta"], t["pairs"])
    kw = dict(s=t["s"], theta=t["theta"], pairs=t["pairs"]) if otf else {}
    y = paro.paro_linear(t["x"], pk, flags=flags, **kw)
    torch.cuda.synchronize()
    rows = np.arange(min(N, 64))
    ref = O.oracle_pack(p["W"][rows], p["s"], p["theta"], p["pairs"])
    y_ref = O.oracle_linear(p["x"], ref, p["s"], p["theta"], p["pairs"])
    err = O.normwise_error(y.float().cpu().numpy()[:, rows], y_ref)
    print(f"N={N} K={K} B={B} flags={flags:#x} otf={otf}: err {err:.2e}", flush=True)
    assert err < 2e-3


def multi():
    K = 1024
    ps = [synth.make_problem(N, K, 1, seed=10 + i) for i, N in enumerate((512, 128, 256))]
    pks = []
    for p in ps:
        t = dev(p)
        pks.append(paro.paro_pack(t["W"], t["s"], t["theta"], t["pairs"]))
    ys = paro.paro_linear_multi(torch.from_numpy(ps[0]["x"]).cuda(), pks)
    torch.cuda.synchronize()
    for p, y in zip(ps, ys):
        ref = O.oracle_pack(p["W"], p["s"], p["theta"], p["pairs"])
        y_ref = O.oracle_linear(ps[0]["x"], ref, p["s"], p["theta"], p["pairs"])
        assert O.normwise_error(y.float().cpu().numpy(), y_ref) < 2e-3
    print("multi ok", flush=True)


def chain(B):
    """Two dependent stages in one persistent launch (grid barrier; B > 1: in-kernel transform)."""
    pa = synth.make_problem(256, 512, B, seed=20)
    pb = synth.make_problem(128, 256, B, seed=21)
    ta, tb = dev(pa), dev(pb)
    ka = paro.paro_pack(ta["W"], ta["s"], ta["theta"], ta["pairs"])
    kb = paro.paro_pack(tb["W"], tb["s"], tb["theta"], tb["pairs"])
    y0 = torch.empty((B, 256), dtype=torch.float16, device="cuda")
    y1 = torch.empty((B, 128), dtype=torch.float16, device="cuda")
    paro.paro_linear_chain([paro.ChainStage(ta["x"], [ka], [y0]), paro.ChainStage(y0, [kb], [y1])])
    torch.cuda.synchronize()
    ra = O.oracle_pack(pa["W"], pa["s"], pa["theta"], pa["pairs"])
    rb = O.oracle_pack(pb["W"], pb["s"], pb["theta"], pb["pairs"])
    assert O.normwise_error(y0.float().cpu().numpy(), O.oracle_linear(pa["x"], ra, pa["s"], pa["theta"], pa["pairs"])) < 2e-3
    y0n = y0.float().cpu().numpy()
    assert O.normwise_error(y1.float().cpu().numpy(), O.oracle_linear(y0n, rb, pb["s"], pb["theta"], pb["pairs"])) < 2e-3
    print(f"chain B={B} ok", flush=True)


def dense(B=130, K=1024):
    """Prefill-form transform: M rows by the Givens kernel on unit vectors, tcgen05 contraction."""
    p = synth.make_problem(8, K, B, seed=30)
    t = dev(p)
    pk = paro.paro_pack(t["W"], t["s"], t["theta"], t["pairs"])
    xp = paro.paro_transform_activations_dense(t["x"], pk).float().cpu().numpy()
    ref = O.transform_activations(p["x"], p["s"], p["theta"], p["pairs"])
    assert np.max(np.abs(xp - ref)) <= 2e-3 * np.max(np.abs(ref))
    print("dense ok", flush=True)


def copy():
    """paro_copy: pinned host -> device -> pinned host, PDL-chained."""
    src = torch.arange(4096 * 3, dtype=torch.int32).pin_memory()
    d = torch.empty(src.shape, dtype=torch.int32, device="cuda")
    back = torch.empty_like(src).pin_memory()
    paro.paro_copy(d, src, flags=paro.PARO_LINEAR_PDL)
    paro.paro_copy(back, d, flags=paro.PARO_LINEAR_PDL)
    torch.cuda.synchronize()
    assert torch.equal(back, src)
    print("copy ok", flush=True)


CASES = {
    "dense": dense,
    "copy": copy,
    "c1": lambda: case(256, 256, 1),
    "q_b1_pdl": lambda: case(1024, 4096, 1, paro.PARO_LINEAR_PDL),
    "q_b3": lambda: case(1024, 4096, 3),
    "q_b2": lambda: case(1024, 4096, 2),
    "q_b16": lambda: case(1024, 4096, 16),
    "otf_b5": lambda: case(512, 1024, 5, otf=True),
    "otf_b1": lambda: case(512, 1024, 1, otf=True),
    "prefill_b300": lambda: case(256, 512, 300, paro.PARO_LINEAR_FORCE_GEMM),
    "multi": multi,
    "chain_b1": lambda: chain(1),
    "chain_b4": lambda: chain(4),
    "q_b8_tcgen05": lambda: case(1024, 4096, 8, paro.PARO_LINEAR_TCGEN05),
}


def main():
    names = [a for a in sys.argv[1:] if not a.startswith("--")] or list(CASES)
    for n in names:
        CASES[n]()
    print("SANITIZE CASES DONE", flush=True)


if __name__ == "__main__":
    main()
