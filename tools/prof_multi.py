"""Launch one decode group (linears sharing x) a few times, for ncu.
argv: Ns (comma list, e.g. 4096,1024,1024) K (rot|norot) reps"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_10645_b200 as paro  # noqa: E402
import synth  # noqa: E402

Ns = [int(v) for v in sys.argv[1].split(",")]
K, mode, reps = int(sys.argv[2]), sys.argv[3], int(sys.argv[4])
B = int(sys.argv[5]) if len(sys.argv) > 5 else 1
flags = paro.PARO_LINEAR_TCGEN05 if (len(sys.argv) > 6 and sys.argv[6] == "tc") else 0
dev = torch.device("cuda")
p = synth.make_problem(8, K, 1, seed=1)
s, th, pr = (torch.from_numpy(p[k]).to(dev) for k in ("s", "theta", "pairs"))
# two weight sets so consecutive launches do not hit L2
sets = [[paro.paro_pack((torch.randn(N, K, device=dev) * 0.02).half(), s, th, pr) for N in Ns] for _ in range(2)]
x = torch.randn(B, K, device=dev).half()
fl = (paro.PARO_LINEAR_NO_ROTATION if mode == "norot" else 0) | flags
for r in range(reps):
    ys = paro.paro_linear_multi(x, sets[r % 2], flags=fl)
torch.cuda.synchronize()
print("ok")
