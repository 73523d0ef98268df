"""Decode GEMV on L2-resident weights (same packed linear every launch): compute-side
throughput ceiling.  argv: N K [reps] [rot|norot]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_10645_b200 as paro  # noqa: E402
import synth  # noqa: E402

N, K = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 100
mode = sys.argv[4] if len(sys.argv) > 4 else "rot"
dev = torch.device("cuda")
p = synth.make_problem(8, K, 1, seed=1)
s, th, pr = (torch.from_numpy(p[k]).to(dev) for k in ("s", "theta", "pairs"))
pk = paro.paro_pack((torch.randn(N, K, device=dev) * 0.02).half(), s, th, pr)
x = torch.randn(1, K, device=dev).half()
y = torch.empty(1, N, device=dev).half()
fl = paro.PARO_LINEAR_NO_ROTATION if mode == "norot" else 0
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    for _ in range(3):
        paro.paro_linear(x, pk, y=y, flags=fl, stream=st)
    st.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(reps):
            paro.paro_linear(x, pk, y=y, flags=fl, stream=st)
    g.replay()
    st.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    g.replay()
    e1.record(st)
    e1.synchronize()
us = e0.elapsed_time(e1) / reps * 1000
b = N * K * 0.5195
print(f"L2-resident {mode} N={N} K={K}: {us:.2f} us/launch  {b / us / 1e3:.0f} GB/s")
