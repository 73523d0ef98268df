"""Graph timing of the bench's launch groups (q/k/v, o, gate/up, down) at bs=1, weight
pool > L2.  argv: [rot|norot] [pdl]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_10645_b200 as paro  # noqa: E402
import synth  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "rot"
pdl = int(sys.argv[2]) if len(sys.argv) > 2 else 1
dev = torch.device("cuda")
shapes = synth.LLAMA3_8B_DECODE
groups = [["q_proj", "k_proj", "v_proj"], ["o_proj"], ["gate_proj", "up_proj"], ["down_proj"]]
prm = {}
for name, (N, K) in shapes.items():
    if K not in prm:
        p = synth.make_problem(8, K, 1, seed=1)
        prm[K] = tuple(torch.from_numpy(p[k]).to(dev) for k in ("s", "theta", "pairs"))
npool = 5
pool = []
for li in range(npool):
    d = {}
    for name, (N, K) in shapes.items():
        s, th, pr = prm[K]
        d[name] = paro.paro_pack((torch.randn(N, K, device=dev) * 0.02).half(), s, th, pr)
    pool.append(d)
xs = {K: torch.randn(1, K, device=dev).half() for K in prm}
ys = {name: torch.empty(1, N, device=dev, dtype=torch.half) for name, (N, K) in shapes.items()}
flags = (paro.PARO_LINEAR_NO_ROTATION if mode == "norot" else 0) | (paro.PARO_LINEAR_PDL if pdl else 0)
st = torch.cuda.Stream()
reps = 50
for grp in groups + [sum(groups, [])]:
    g = torch.cuda.CUDAGraph()
    K = shapes[grp[0]][1]

    def run(i):
        if len(grp) > 4:
            for gg in groups:
                KK = shapes[gg[0]][1]
                paro.paro_linear_multi(xs[KK], [pool[i % npool][n] for n in gg], y=[ys[n] for n in gg], flags=flags,
                                       stream=st)
        else:
            paro.paro_linear_multi(xs[K], [pool[i % npool][n] for n in grp], y=[ys[n] for n in grp], flags=flags,
                                   stream=st)

    with torch.cuda.stream(st):
        run(0)
        st.synchronize()
        with torch.cuda.graph(g, stream=st):
            for i in range(reps):
                run(i)
        g.replay()
        st.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(3):
            g.replay()
        e1.record(st)
    e1.synchronize()
    us = e0.elapsed_time(e1) / (3 * reps) * 1e3
    nbytes = sum(shapes[n][0] * shapes[n][1] * 0.5195 for n in (grp if len(grp) <= 4 else sum(groups, [])))
    print(f"{mode} pdl={pdl} {'+'.join(grp) if len(grp) <= 4 else 'layer'}: {us:.2f} us  {nbytes / us / 1e3:.0f} GB/s")
