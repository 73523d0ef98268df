"""Prefill (2048 tokens) per LLaMA-3-8B linear: total paro_linear (transform pre-stage + tcgen05
GEMM), the transform alone (paro_transform_activations) and TFLOP/s; argv[1]: package dir."""
import os
import sys

sys.path.insert(0, os.path.abspath(sys.argv[1] if len(sys.argv) > 1 else "."))
sys.path.insert(1, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2511_10645_b200 as paro  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda")
st = torch.cuda.Stream()


def t_us(fn, reps=10):
    with torch.cuda.stream(st):
        fn()
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(reps):
                fn()
        g.replay()
        st.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        g.replay()
        e1.record(st)
        e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


Bp = 2048
tot_f, tot_us = 0.0, 0.0
for name, (N, K) in synth.LLAMA3_8B_DECODE.items():
    p = synth.make_problem(8, K, 1, seed=N % 97)
    s, th, pr = (torch.from_numpy(p[k]).to(dev) for k in ("s", "theta", "pairs"))
    pk = paro.paro_pack((torch.randn(N, K, device=dev) * 0.02).half(), s, th, pr)
    x = torch.randn(Bp, K, device=dev).half()
    y = torch.empty(Bp, N, device=dev, dtype=torch.half)
    xo = torch.empty(Bp, K, device=dev, dtype=torch.half)
    ws = torch.empty(max(1, paro.paro_linear_workspace(Bp, N, K)), dtype=torch.uint8, device=dev)
    us = t_us(lambda: paro.paro_linear(x, pk, y=y, workspace=ws, stream=st))
    ut = t_us(lambda: paro.paro_transform_activations(x, pk, out=xo, stream=st))
    f = 2.0 * Bp * N * K
    tot_f += f
    tot_us += us
    print(f"{name:10s} N={N:6d} K={K:6d}: total {us:7.2f} us ({f / us / 1e6:6.1f} TF/s)  transform {ut:6.2f} us  "
          f"GEMM ~{us - ut:7.2f} us ({f / (us - ut) / 1e6:6.1f} TF/s)", flush=True)
print(f"layer: {tot_us:.1f} us, {tot_f / tot_us / 1e6:.1f} TFLOP/s", flush=True)
