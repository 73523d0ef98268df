"""Standalone activation transform timing (rotation kernel microbenchmark,
fig:kernel-speedup's 'our transform'): argv K B"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_10645_b200 as paro  # noqa: E402
import synth  # noqa: E402

K, B = int(sys.argv[1]), int(sys.argv[2])
dev = torch.device("cuda")
p = synth.make_problem(8, K, 1, seed=1)
s, th, pr = (torch.from_numpy(p[k]).to(dev) for k in ("s", "theta", "pairs"))
pk = paro.paro_pack((torch.randn(128, K, device=dev) * 0.02).half(), s, th, pr)
x = torch.randn(B, K, device=dev).half()
out = torch.empty_like(x)
for _ in range(3):
    paro.paro_transform_activations(x, pk, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    paro.paro_transform_activations(x, pk, out=out)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 20 * 1e3
print(f"transform K={K} B={B}: {us:.2f} us  {B * K * 4 / us / 1e3:.0f} GB/s  {B * K / 128 / us:.1f} group-items/us")
