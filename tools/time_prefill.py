"""Prefill (tcgen05 GEMM + transform pre-stage) timing at B tokens for the LLaMA-3-8B shapes.
argv: [B]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_10645_b200 as paro  # noqa: E402
import synth  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
dev = torch.device("cuda")
st = torch.cuda.Stream()
tot_flop, tot_us = 0.0, 0.0
for name, (N, K) in synth.LLAMA3_8B_DECODE.items():
    p = synth.make_problem(8, K, 1, seed=1)
    s, th, pr = (torch.from_numpy(p[k]).to(dev) for k in ("s", "theta", "pairs"))
    pk = paro.paro_pack((torch.randn(N, K, device=dev) * 0.02).half(), s, th, pr)
    x = torch.randn(B, K, device=dev).half()
    y = torch.empty(B, N, device=dev).half()
    ws = torch.empty(paro.paro_linear_workspace(B, N, K), dtype=torch.uint8, device=dev)
    with torch.cuda.stream(st):
        for _ in range(3):
            paro.paro_linear(x, pk, y=y, workspace=ws, stream=st)
        reps = 20
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(reps):
                paro.paro_linear(x, pk, y=y, workspace=ws, stream=st)
        g.replay()
        st.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        g.replay()
        e1.record(st)
        e1.synchronize()
    us = e0.elapsed_time(e1) / reps * 1000
    fl = 2.0 * B * N * K
    tot_flop += fl
    tot_us += us
    print(f"{name}: B={B} N={N} K={K}: {us:.1f} us  {fl / us / 1e6:.1f} TFLOP/s")
print(f"layer: {tot_us:.1f} us  {tot_flop / tot_us / 1e6:.1f} TFLOP/s")
