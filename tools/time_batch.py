"""Decode launch time vs token count (graph of reps calls over 2 weight sets).  argv: N K [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_10645_b200 as paro  # noqa: E402
import synth  # noqa: E402

N, K = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 50
dev = torch.device("cuda")
p = synth.make_problem(8, K, 1, seed=1)
s, th, pr = (torch.from_numpy(p[k]).to(dev) for k in ("s", "theta", "pairs"))
sets = [paro.paro_pack((torch.randn(N, K, device=dev) * 0.02).half(), s, th, pr) for _ in range(4)]
st = torch.cuda.Stream()
for B in (int(v) for v in os.environ.get("TB_BATCHES", "1,2,4,8,16").split(",")):
    x = torch.randn(B, K, device=dev).half()
    y = torch.empty(B, N, device=dev).half()
    with torch.cuda.stream(st):
        for i in range(2):
            paro.paro_linear(x, sets[i], y=y, flags=paro.PARO_LINEAR_PDL, stream=st)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for i in range(reps):
                paro.paro_linear(x, sets[i % 4], y=y, flags=paro.PARO_LINEAR_PDL, stream=st)
        g.replay()
        st.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        g.replay()
        e1.record(st)
        e1.synchronize()
    us = e0.elapsed_time(e1) / reps * 1e3
    print(f"N={N} K={K} B={B}: {us:.2f} us/call  {N * K * 0.5195 / us / 1e3:.0f} GB/s")
