"""One prefill shape a few times (for ncu): argv N K B [reps]."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_10645_b200 as paro  # noqa: E402
import synth  # noqa: E402

N, K, B = (int(v) for v in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
dev = torch.device("cuda")
p = synth.make_problem(8, K, 1, seed=1)
s, th, pr = (torch.from_numpy(p[k]).to(dev) for k in ("s", "theta", "pairs"))
pk = paro.paro_pack((torch.randn(N, K, device=dev) * 0.02).half(), s, th, pr)
x = torch.randn(B, K, device=dev).half()
ws = torch.empty(paro.paro_linear_workspace(B, N, K), dtype=torch.uint8, device=dev)
for _ in range(reps):
    y = paro.paro_linear(x, pk, workspace=ws)
torch.cuda.synchronize()
print("ok")
