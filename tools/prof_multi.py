"""Launch the gate/up pair (or any N x n_lin at K) a few times for ncu.  argv: N K n_lin (rot|norot) reps"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_10645_b200 as paro  # noqa: E402
import synth  # noqa: E402

N, K, n, mode, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], int(sys.argv[5])
dev = torch.device("cuda")
p = synth.make_problem(8, K, 1, seed=1)
s, th, pr = (torch.from_numpy(p[k]).to(dev) for k in ("s", "theta", "pairs"))
pks = [paro.paro_pack((torch.randn(N, K, device=dev) * 0.02).half(), s, th, pr) for _ in range(n)]
x = torch.randn(1, K, device=dev).half()
fl = paro.PARO_LINEAR_NO_ROTATION if mode == "norot" else 0
for _ in range(reps):
    ys = paro.paro_linear_multi(x, pks, flags=fl)
torch.cuda.synchronize()
print("ok")
