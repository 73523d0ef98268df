"""One B > 1 decode multi-launch shape, repeated (for ncu): argv[1] B, argv[2] 'qkv'|'gateup'|'down'
(Qwen3-4B shapes, K = 2560 / 9728)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2511_10645_b200 as paro  # noqa: E402
import synth  # noqa: E402

B = int(sys.argv[1])
which = sys.argv[2]
Ns, K = {"qkv": ([4096, 1024, 1024], 2560), "gateup": ([9728, 9728], 2560), "down": ([2560], 9728)}[which]
dev = torch.device("cuda")
p = synth.make_problem(8, K, 1, seed=3)
s, th, pr = (torch.from_numpy(p[k]).to(dev) for k in ("s", "theta", "pairs"))
pool = [[paro.paro_pack((torch.randn(N, K, device=dev) * 0.02).half(), s, th, pr) for N in Ns] for _ in range(6)]
x = torch.randn(B, K, device=dev).half()
ys = [torch.empty(B, N, device=dev, dtype=torch.half) for N in Ns]
ws = torch.empty(64 << 20, dtype=torch.uint8, device=dev)
for i in range(30):
    paro.paro_linear_multi(x, pool[i % 6], y=ys, flags=paro.PARO_LINEAR_PDL, workspace=ws)
torch.cuda.synchronize()
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for i in range(20):
            paro.paro_linear_multi(x, pool[i % 6], y=ys, flags=paro.PARO_LINEAR_PDL, workspace=ws, stream=st)
    g.replay()
    st.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    g.replay()
    e1.record(st)
    e1.synchronize()
print(f"B={B} {which}: {e0.elapsed_time(e1) / 20 * 1e3:.2f} us per launch (graph of 20)", flush=True)
