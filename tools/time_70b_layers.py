"""LLaMA-3-70B gate_proj (28672 x 8192) at bs=1: time vs the number of rotation layers L packed
(0, 1, 2, 4, 8) and with rotation disabled -- separates per-layer cost (tables, rotations) from the
scale / transform skeleton.  Graph of 20 PDL calls over two weight copies."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_10645_b200 as paro  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda")
st = torch.cuda.Stream()
N, K = int(sys.argv[1]) if len(sys.argv) > 1 else 28672, int(sys.argv[2]) if len(sys.argv) > 2 else 8192


def timed(pks, x, y, fl):
    with torch.cuda.stream(st):
        for i in range(2):
            paro.paro_linear(x, pks[i], y=y, flags=fl | paro.PARO_LINEAR_PDL, stream=st)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for i in range(20):
                paro.paro_linear(x, pks[i % 2], y=y, flags=fl | paro.PARO_LINEAR_PDL, stream=st)
        g.replay()
        st.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        g.replay()
        e1.record(st)
        e1.synchronize()
    return e0.elapsed_time(e1) / 20 * 1e3


x = torch.randn(1, K, device=dev).half()
y = torch.empty(1, N, device=dev).half()
for L in (0, 1, 2, 4, 8):
    p = synth.make_problem(8, K, 1, seed=3, n_rot=L)
    s, th, pr = (torch.from_numpy(p[k]).to(dev) for k in ("s", "theta", "pairs"))
    pks = [paro.paro_pack((torch.randn(N, K, device=dev) * 0.02).half(), s, th, pr) for _ in range(2)]
    r = timed(pks, x, y, 0)
    nr = timed(pks, x, y, paro.PARO_LINEAR_NO_ROTATION)
    print(f"N={N} K={K} L={L}: {r:.2f} us (rotation disabled: {nr:.2f})", flush=True)
    del pks
