"""A/B: the LLaMA-3-8B decode step as 4 PDL-chained paro_linear_multi launches (and per-linear
single launches) with the package found first on sys.path (argv[1]: a directory containing
paper_2511_10645_b200), pool of 5 layers (> 4 x L2), CUDA graph of 20 steps, CUDA events."""
import os
import sys

sys.path.insert(0, os.path.abspath(sys.argv[1]))
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(1, ROOT)
import torch  # noqa: E402

import paper_2511_10645_b200 as paro  # noqa: E402
import synth  # noqa: E402

print("package", paro.__file__, flush=True)
dev = torch.device("cuda")
shapes = synth.LLAMA3_8B_DECODE
G_cache = {}
pool = []
for li in range(5):
    layer = {}
    for name, (N, K) in shapes.items():
        if (N, K) not in G_cache:
            p = synth.make_problem(8, K, 1, seed=N % 97)
            G_cache[(N, K)] = tuple(torch.from_numpy(p[k]).to(dev) for k in ("s", "theta", "pairs"))
        s, th, pr = G_cache[(N, K)]
        W = (torch.randn((N, K), device=dev) * 0.02).half()
        layer[name] = paro.paro_pack(W, s, th, pr)
    pool.append(layer)
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
XF = paro.PARO_LINEAR_TCGEN05 if (len(sys.argv) > 3 and sys.argv[3] == "tc") else 0
x = torch.randn(B, 4096, device=dev).half()
x2 = torch.randn(B, 14336, device=dev).half()
ys = {n: torch.empty(B, N, device=dev, dtype=torch.half) for n, (N, K) in shapes.items()}
ws = torch.empty(64 << 20, dtype=torch.uint8, device=dev)
groups = [["q_proj", "k_proj", "v_proj"], ["o_proj"], ["gate_proj", "up_proj"], ["down_proj"]]
st = torch.cuda.Stream()


def timed(fn, reps=20):
    with torch.cuda.stream(st):
        fn(0)
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for i in range(reps):
                fn(i)
        for _ in range(5):
            g.replay()
        st.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(5):
            e0.record(st)
            g.replay()
            e1.record(st)
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) / reps * 1e3)
    return best


def step(i):
    L = pool[i % 5]
    for grp in groups:
        xin = x2 if grp[0] == "down_proj" else x
        paro.paro_linear_multi(xin, [L[n] for n in grp], y=[ys[n] for n in grp], flags=paro.PARO_LINEAR_PDL | XF,
                               workspace=ws, stream=st)


print(f"B={B} step (4 launches): {timed(step):.2f} us", flush=True)
if hasattr(paro, "paro_linear_chain"):
    chains = []
    for L in pool:
        chains.append([paro.ChainStage(x, [L[n] for n in groups[0]], [ys[n] for n in groups[0]]),
                       paro.ChainStage(x, [L["o_proj"]], [ys["o_proj"]]),
                       paro.ChainStage(x, [L[n] for n in groups[2]], [ys[n] for n in groups[2]]),
                       paro.ChainStage(x2, [L["down_proj"]], [ys["down_proj"]])])
    cws = paro.chain_workspace(B, chains[0])

    def chain_step(i):
        paro.paro_linear_chain(chains[i % 5], flags=paro.PARO_LINEAR_PDL | XF, workspace=cws, stream=st)

    try:
        print(f"B={B} step (chain): {timed(chain_step):.2f} us", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"B={B} step (chain): {e}", flush=True)
for grp in groups:
    def one(i, grp=grp):
        L = pool[i % 5]
        xin = x2 if grp[0] == "down_proj" else x
        paro.paro_linear_multi(xin, [L[n] for n in grp], y=[ys[n] for n in grp], flags=paro.PARO_LINEAR_PDL | XF,
                               workspace=ws, stream=st)
    print(f"{'+'.join(grp)}: {timed(one):.2f} us", flush=True)
