"""B <= 16 tokens: the prefill tcgen05 GEMM (PARO_LINEAR_FORCE_GEMM) vs the decode GEMV, single
linears, graph of 20 PDL-chained calls.  argv: B [N,K ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_10645_b200 as paro  # noqa: E402
import synth  # noqa: E402

B = int(sys.argv[1])
shapes = [tuple(int(v) for v in a.split(",")) for a in sys.argv[2:]] or [(4096, 2560), (9728, 2560), (2560, 9728)]
dev = torch.device("cuda")
st = torch.cuda.Stream()
for N, K in shapes:
    p = synth.make_problem(8, K, 1, seed=1)
    s, th, pr = (torch.from_numpy(p[k]).to(dev) for k in ("s", "theta", "pairs"))
    pool = [paro.paro_pack((torch.randn(N, K, device=dev) * 0.02).half(), s, th, pr) for _ in range(6)]
    x = torch.randn(B, K, device=dev).half()
    y = torch.empty(B, N, device=dev).half()
    res = {}
    for name, fl in (("gemv", 0), ("gemm", paro.PARO_LINEAR_FORCE_GEMM)):
        ws = torch.empty(paro.paro_linear_workspace(B, N, K, flags=fl), dtype=torch.uint8, device=dev)
        with torch.cuda.stream(st):
            for i in range(3):
                paro.paro_linear(x, pool[i % 6], y=y, flags=fl | paro.PARO_LINEAR_PDL, workspace=ws, stream=st)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                for i in range(20):
                    paro.paro_linear(x, pool[i % 6], y=y, flags=fl | paro.PARO_LINEAR_PDL, workspace=ws, stream=st)
            g.replay()
            st.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            g.replay()
            e1.record(st)
            e1.synchronize()
        res[name] = e0.elapsed_time(e1) / 20 * 1e3
    print(f"B={B} N={N} K={K}: gemv {res['gemv']:.2f} us, gemm {res['gemm']:.2f} us", flush=True)
