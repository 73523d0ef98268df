"""Dense transform (paro_transform_activations_dense) at T tokens x n channels, repeated (ncu driver).
argv: n T"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2511_10645_b200 as paro  # noqa: E402
import synth  # noqa: E402

n, T = int(sys.argv[1]), int(sys.argv[2])
dev = torch.device("cuda")
p = synth.make_problem(32, n, 1, seed=n)
t = {k: torch.from_numpy(p[k]).to(dev) for k in ("W", "s", "theta", "pairs")}
packed = paro.paro_pack(t["W"], t["s"], t["theta"], t["pairs"])
x = torch.randn((T, n), device=dev).to(torch.float16)
y = torch.empty_like(x)
ws = torch.empty(paro._lib.paro_transform_dense_workspace(n), dtype=torch.uint8, device=dev)
for _ in range(5):
    paro.paro_transform_activations_dense(x, packed, out=y, workspace=ws)
    paro.paro_transform_activations(x, packed, out=y)
torch.cuda.synchronize()
