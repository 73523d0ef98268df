"""Debug: one decode linear at B > 1 (tcgen05 path) and a 2-stage chain, small shapes."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2511_10645_b200 as paro  # noqa: E402
import synth  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 3
mode = sys.argv[2] if len(sys.argv) > 2 else "single"
N, K = 256, 512
p = synth.make_problem(N, K, B, seed=1)
t = {k: torch.from_numpy(p[k]).cuda() for k in ("W", "s", "theta", "pairs", "x")}
pk = paro.paro_pack(t["W"], t["s"], t["theta"], t["pairs"])
ref = O.oracle_pack(p["W"], p["s"], p["theta"], p["pairs"])
yref = O.oracle_linear(p["x"], ref, p["s"], p["theta"], p["pairs"])
if mode == "single":
    y = paro.paro_linear(t["x"], pk)
else:
    y = torch.empty((B, N), dtype=torch.float16, device="cuda")
    y2 = torch.empty((B, N), dtype=torch.float16, device="cuda")
    paro.paro_linear_chain([paro.ChainStage(t["x"], [pk], [y]), paro.ChainStage(t["x"], [pk], [y2])])
torch.cuda.synchronize()
print(f"B={B} {mode}: err {O.normwise_error(y.float().cpu().numpy(), yref):.3e}", flush=True)
