"""Per-CTA event timeline of the last decode (B=1) launch of a CUDA graph of PDL launches
(needs a library built with PARO_NVCC_EXTRA=-DG1_TL=1).  argv: Ns(comma) K (rot|norot)"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("PARO_PKG_DIR"):
    sys.path.insert(0, os.path.abspath(os.environ["PARO_PKG_DIR"]))
import paper_2511_10645_b200 as paro  # noqa: E402
import synth  # noqa: E402

Ns = [int(v) for v in sys.argv[1].split(",")]
K, mode = int(sys.argv[2]), sys.argv[3]
dev = torch.device("cuda")
p = synth.make_problem(8, K, 1, seed=1)
s, th, pr = (torch.from_numpy(p[k]).to(dev) for k in ("s", "theta", "pairs"))
npool = max(2, int(600e6 / (sum(Ns) * K * 0.52)))
npool = min(npool, 12)
pool = [[paro.paro_pack((torch.randn(N, K, device=dev) * 0.02).half(), s, th, pr) for N in Ns] for _ in range(npool)]
x = torch.randn(1, K, device=dev).half()
ys = [torch.empty(1, N, device=dev, dtype=torch.half) for N in Ns]
fl = (paro.PARO_LINEAR_NO_ROTATION if mode == "norot" else 0) | paro.PARO_LINEAR_PDL
st = torch.cuda.Stream()
reps = 20
with torch.cuda.stream(st):
    paro.paro_linear_multi(x, pool[0], y=ys, flags=fl, stream=st)
    st.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for i in range(reps):
            paro.paro_linear_multi(x, pool[i % npool], y=ys, flags=fl, stream=st)
    for _ in range(3):
        g.replay()
    st.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    g.replay()
    e1.record(st)
e1.synchronize()
print(f"{sys.argv[1]} K={K} {mode}: {e0.elapsed_time(e1) / reps * 1e3:.2f} us per launch (graph, PDL)")
lib = paro._lib
lib.paro_debug_read_timeline1.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros(1024 * 12, dtype=np.uint64)
lib.paro_debug_read_timeline1(buf.ctypes.data, buf.size)
t = buf.reshape(1024, 12).astype(np.int64)
live = t[:, 0] > 0
t = t[live]
rel = (t - t[:, 0].min()) / 1000.0
names = ["start", "all_issued(prod)", "x_arrived", "transform_done", "stage0_ready", "tiles_done", "reduced", "end",
         "w0_layer0_done", "w0_rotations_done"]
for i, n in enumerate(names):
    col = rel[:, i]
    print(f"  {n:18s} min {col.min():7.2f}  median {np.median(col):7.2f}  max {col.max():7.2f}")
