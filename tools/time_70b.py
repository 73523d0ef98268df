"""LLaMA-3-70B MLP decode launches (gate+up fused, down) at bs=1: graph of PDL calls over two
weight copies.  Env PARO_G1_CL etc. select the plan."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_10645_b200 as paro  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda")
shapes = synth.LLAMA3_70B_MLP
prm = {}
sets = []
for li in range(2):
    d = {}
    for name, (N, K) in shapes.items():
        if K not in prm:
            p = synth.make_problem(8, K, 1, seed=3)
            prm[K] = tuple(torch.from_numpy(p[k]).to(dev) for k in ("s", "theta", "pairs"))
        d[name] = paro.paro_pack((torch.randn(N, K, device=dev) * 0.02).half(), *prm[K])
    sets.append(d)
st = torch.cuda.Stream()
for grp in (["gate_proj", "up_proj"], ["down_proj"]):
    K = shapes[grp[0]][1]
    x = torch.randn(1, K, device=dev).half()
    ys = [torch.empty(1, shapes[n][0], device=dev).half() for n in grp]
    reps = 20
    with torch.cuda.stream(st):
        paro.paro_linear_multi(x, [sets[0][n] for n in grp], y=ys, flags=paro.PARO_LINEAR_PDL, stream=st)
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for i in range(reps):
                paro.paro_linear_multi(x, [sets[i % 2][n] for n in grp], y=ys, flags=paro.PARO_LINEAR_PDL, stream=st)
        g.replay()
        st.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        g.replay()
        e1.record(st)
        e1.synchronize()
    us = e0.elapsed_time(e1) / reps * 1e3
    nb = sum(shapes[n][0] * K * 0.5195 for n in grp)
    print(f"{'+'.join(grp)}: {us:.2f} us  {nb / us / 1e3:.0f} GB/s")
