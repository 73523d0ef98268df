"""Launch one decode linear a few times (for ncu): argv = N K (rot|norot) reps [B]."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_10645_b200 as paro  # noqa: E402
import synth  # noqa: E402

N, K = int(sys.argv[1]), int(sys.argv[2])
mode = sys.argv[3] if len(sys.argv) > 3 else "rot"
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
B = int(sys.argv[5]) if len(sys.argv) > 5 else 1
p = synth.make_problem(8, K, 1, seed=1)
dev = torch.device("cuda")
s, th, pr = (torch.from_numpy(p[k]).to(dev) for k in ("s", "theta", "pairs"))
W = (torch.randn(N, K, device=dev) * 0.02).half()
pk = paro.paro_pack(W, s, th, pr)
x = torch.randn(B, K, device=dev).half()
flags = paro.PARO_LINEAR_NO_ROTATION if mode == "norot" else 0
y = paro.paro_linear(x, pk, flags=flags)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    paro.paro_linear(x, pk, y=y, flags=flags)
e1.record()
torch.cuda.synchronize()
print(f"N={N} K={K} B={B} {mode}: {e0.elapsed_time(e1) / reps * 1e3:.2f} us/call eager (L2-warm)")
