"""Per-CTA timeline of the LAST launch of a graph of LLaMA-3-8B decode chains (bs=1).  Needs the
library built with PARO_NVCC_EXTRA=-DPARO_TIMELINE=1 (force rebuild).  argv: chain|multi
Events per (CTA, stage): 0 kernel start, 1 x available (PDL / grid barrier), 2 transform done,
3 first batch landed, 4 tiles done, 5 cluster partials in, 6 stores done, 7 producer issued all."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2511_10645_b200 as paro  # noqa: E402
import synth  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "chain"
dev = torch.device("cuda")
shapes = synth.LLAMA3_8B_DECODE
n_layers = 5
pool = bench.build_layer_pool(torch, paro, shapes, 0, 1, n_layers, dev)
x_in = torch.randn(1, 4096, device=dev).half()
x_attn = torch.randn(1, 4096, device=dev).half()
ys = {n: torch.empty(1, N, device=dev, dtype=torch.half) for n, (N, K) in shapes.items()}
chains = [bench.layer_chain(paro, layer, x_in, x_attn, ys) for layer in pool]
ws = paro.chain_workspace(1, chains[0])
st = torch.cuda.Stream()
reps = 10


def step(li):
    if mode == "chain":
        paro.paro_linear_chain(chains[li % n_layers], flags=paro.PARO_LINEAR_PDL, workspace=ws, stream=st)
    else:
        for s in chains[li % n_layers]:
            paro.paro_linear_multi(s.x, s.packed, y=s.y, flags=paro.PARO_LINEAR_PDL, stream=st)


with torch.cuda.stream(st):
    step(0)
    st.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for i in range(reps):
            step(i)
    for _ in range(3):
        g.replay()
    st.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    g.replay()
    e1.record(st)
    e1.synchronize()
print(f"{mode}: {e0.elapsed_time(e1) / reps * 1e3:.2f} us per step", flush=True)
lib = ctypes.CDLL(paro.LIB_PATH)
buf = np.zeros(1024 * 16 * 8, dtype=np.uint64)
lib.paro_debug_timeline(buf.ctypes.data_as(ctypes.c_void_p), buf.size)
tl = buf.reshape(1024, 16, 8).astype(np.int64)
ncta = int((tl[:, 0, 0] > 0).sum())
t0 = tl[:ncta, 0, 0].min()
names = ["start", "x", "xform", "batch0", "tiles", "recv", "stored", "prod"]
nst = 4 if mode == "chain" else 1
for s in range(nst):
    row = []
    for e in range(8):
        v = tl[:ncta, s, e]
        v = v[v > 0]
        if len(v) == 0:
            row.append(f"{names[e]}=-")
            continue
        row.append(f"{names[e]}={(np.median(v) - t0) / 1e3:.2f}[{(v.min() - t0) / 1e3:.2f},{(v.max() - t0) / 1e3:.2f}]")
    print(f"stage {s}: " + " ".join(row), flush=True)
