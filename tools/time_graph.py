"""CUDA-graph timing of one decode linear over a weight pool larger than L2.
argv: N K (rot|norot) [pdl=1] [reps=100] [B=1]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_10645_b200 as paro  # noqa: E402
import synth  # noqa: E402

N, K = int(sys.argv[1]), int(sys.argv[2])
mode = sys.argv[3]
pdl = int(sys.argv[4]) if len(sys.argv) > 4 else 1
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 100
B = int(sys.argv[6]) if len(sys.argv) > 6 else 1
dev = torch.device("cuda")
p = synth.make_problem(8, K, 1, seed=1)
s, th, pr = (torch.from_numpy(p[k]).to(dev) for k in ("s", "theta", "pairs"))
wbytes = N * K // 2
npool = max(2, (4 * 126 * 2**20) // wbytes + 1)
pool = []
for i in range(npool):
    W = (torch.randn(N, K, device=dev) * 0.02).half()
    pool.append(paro.paro_pack(W, s, th, pr))
    del W
x = torch.randn(B, K, device=dev).half()
y = torch.empty(B, N, device=dev, dtype=torch.half)
flags = (paro.PARO_LINEAR_NO_ROTATION if mode == "norot" else 0) | (paro.PARO_LINEAR_PDL if pdl else 0)
st = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(st):
    paro.paro_linear(x, pool[0], y=y, flags=flags, stream=st)
    st.synchronize()
    with torch.cuda.graph(g, stream=st):
        for i in range(reps):
            paro.paro_linear(x, pool[i % npool], y=y, flags=flags, stream=st)
    g.replay()
    st.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(5):
        g.replay()
    e1.record(st)
e1.synchronize()
us = e0.elapsed_time(e1) / (5 * reps) * 1e3
G = K // 128
ab = N * K // 2 + N * G * 2 + N * G // 2
print(f"N={N} K={K} B={B} {mode} pdl={pdl}: {us:.3f} us/launch  {ab / us / 1e3:.0f} GB/s (weights)  pool={npool}")
