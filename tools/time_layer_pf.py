"""LLaMA-3-8B decode layer (4 launches, bs=1, pool of 5 layers > L2) in one CUDA graph with PDL,
with and without the L2 prefetch of the next launch's weights (paro_linear_multi_prefetch).
argv: [prefetch_MB ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_10645_b200 as paro  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda")
shapes = synth.LLAMA3_8B_DECODE
groups = [["q_proj", "k_proj", "v_proj"], ["o_proj"], ["gate_proj", "up_proj"], ["down_proj"]]
prm = {}
for name, (N, K) in shapes.items():
    if K not in prm:
        p = synth.make_problem(8, K, 1, seed=1)
        prm[K] = tuple(torch.from_numpy(p[k]).to(dev) for k in ("s", "theta", "pairs"))
npool = 5
pool = [{name: paro.paro_pack((torch.randn(N, K, device=dev) * 0.02).half(), *prm[K]) for name, (N, K) in shapes.items()}
        for _ in range(npool)]
xs = {K: torch.randn(1, K, device=dev).half() for K in prm}
ys = {name: torch.empty(1, N, device=dev, dtype=torch.half) for name, (N, K) in shapes.items()}
st = torch.cuda.Stream()
reps = 20
seq = [(li, gi) for li in range(reps) for gi in range(len(groups))]
for mb in [0] + [int(v) for v in sys.argv[1:]]:
    def run():
        for idx, (li, gi) in enumerate(seq):
            grp = groups[gi]
            K = shapes[grp[0]][1]
            layer = pool[li % npool]
            nli, ngi = seq[(idx + 1) % len(seq)]
            nxt = [pool[nli % npool][n] for n in groups[ngi]] if mb > 0 else None
            paro.paro_linear_multi(xs[K], [layer[n] for n in grp], y=[ys[n] for n in grp], flags=paro.PARO_LINEAR_PDL,
                                   stream=st, prefetch_next=nxt, prefetch_bytes=mb << 20)
    with torch.cuda.stream(st):
        run()
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            run()
        g.replay()
        st.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(3):
            g.replay()
        e1.record(st)
    e1.synchronize()
    us = e0.elapsed_time(e1) / (3 * reps) * 1e3
    print(f"prefetch {mb} MB: layer {us:.2f} us")
