"""LLaMA-3-70B MLP linears one call at a time (as bench.py's C5 at world 1), rotation on / off,
graph of 20 PDL calls over two weight copies.  Env PARO_G1_CL etc. (debug-knob builds) select the plan."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_10645_b200 as paro  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda")
st = torch.cuda.Stream()
for name, (N, K) in synth.LLAMA3_70B_MLP.items():
    p = synth.make_problem(8, K, 1, seed=3)
    s, th, pr = (torch.from_numpy(p[k]).to(dev) for k in ("s", "theta", "pairs"))
    pks = [paro.paro_pack((torch.randn(N, K, device=dev) * 0.02).half(), s, th, pr) for _ in range(2)]
    x = torch.randn(1, K, device=dev).half()
    y = torch.empty(1, N, device=dev).half()
    res = {}
    for tag, fl in (("rot", 0), ("norot", paro.PARO_LINEAR_NO_ROTATION)):
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
        res[tag] = e0.elapsed_time(e1) / 20 * 1e3
    print(f"{name} N={N} K={K}: {res['rot']:.2f} us (no rotation {res['norot']:.2f}, overhead "
          f"{res['rot'] / res['norot'] - 1:.3f})", flush=True)
    del pks
