"""One decode launch shape, repeated (for ncu): argv[1] package dir, argv[2] 'qkv'|'o'|'gateup'."""
import os
import sys

sys.path.insert(0, os.path.abspath(sys.argv[1]))
sys.path.insert(1, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2511_10645_b200 as paro  # noqa: E402
import synth  # noqa: E402

which = sys.argv[2]
Ns = {"qkv": [4096, 1024, 1024], "o": [4096], "gateup": [14336, 14336]}[which]
K = 4096
dev = torch.device("cuda")
p = synth.make_problem(8, K, 1, seed=3)
s, th, pr = (torch.from_numpy(p[k]).to(dev) for k in ("s", "theta", "pairs"))
pool = [[paro.paro_pack((torch.randn(N, K, device=dev) * 0.02).half(), s, th, pr) for N in Ns] for _ in range(6)]
x = torch.randn(1, K, device=dev).half()
ys = [torch.empty(1, N, device=dev, dtype=torch.half) for N in Ns]
for i in range(30):
    paro.paro_linear_multi(x, pool[i % 6], y=ys, flags=paro.PARO_LINEAR_PDL)
torch.cuda.synchronize()
