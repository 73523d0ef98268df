"""Timeline (PARO_TIMELINE build) of the last of 20 graph-captured launches of one multi-linear
decode launch.  argv: Ns(comma) K B"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_10645_b200 as paro  # noqa: E402
import synth  # noqa: E402

Ns = [int(v) for v in sys.argv[1].split(",")]
K, B = int(sys.argv[2]), int(sys.argv[3])
dev = torch.device("cuda")
p = synth.make_problem(8, K, 1, seed=1)
s, th, pr = (torch.from_numpy(p[k]).to(dev) for k in ("s", "theta", "pairs"))
pool = [[paro.paro_pack((torch.randn(N, K, device=dev) * 0.02).half(), s, th, pr) for N in Ns] for _ in range(6)]
x = torch.randn(B, K, device=dev).half()
ys = [torch.empty(B, N, device=dev, dtype=torch.half) for N in Ns]
ws = torch.empty(64 << 20, dtype=torch.uint8, device=dev)
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    paro.paro_linear_multi(x, pool[0], y=ys, flags=paro.PARO_LINEAR_PDL, workspace=ws, stream=st)
    st.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for i in range(20):
            paro.paro_linear_multi(x, pool[i % 6], y=ys, flags=paro.PARO_LINEAR_PDL, workspace=ws, stream=st)
    g.replay()
    st.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    g.replay()
    e1.record(st)
    e1.synchronize()
print(f"Ns={Ns} K={K} B={B}: {e0.elapsed_time(e1) / 20 * 1e3:.2f} us per launch", flush=True)
lib = ctypes.CDLL(paro.LIB_PATH)
buf = np.zeros(1024 * 16 * 8, dtype=np.uint64)
lib.paro_debug_timeline(buf.ctypes.data_as(ctypes.c_void_p), buf.size)
tl = buf.reshape(1024, 16, 8).astype(np.int64)[:, 0, :]
ncta = int((tl[:, 0] > 0).sum())
tl = tl[:ncta]
t0 = tl[:, 0].min()
names = ["start", "x", "xform", "batch0", "tiles", "recv", "stored", "prod"]
row = []
for e in range(8):
    v = tl[:, e]
    v = v[v > 0]
    if len(v):
        row.append(f"{names[e]}={(np.median(v) - t0) / 1e3:.2f}[{(v.min() - t0) / 1e3:.2f},{(v.max() - t0) / 1e3:.2f}]")
print(" ".join(row), flush=True)
cy = buf.reshape(1024, 16, 8).astype(np.int64)[:ncta, 15, :]
if cy[:, 5].sum() > 0:
    n = cy[:, 5].astype(np.float64)
    print("UMMA item cycles (warp 0, mean per item): fill %.0f  st+wait %.0f  bar %.0f  mma-wait %.0f  ld+epi %.0f  (items/CTA %.1f)"
          % tuple(list((cy[:, :5].sum(axis=0) / n.sum())) + [n.mean()]))
