"""Prefill GEMM MMA-issuer wait profile (library built with -DPARO_PF_PROF=1): argv N K B."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_10645_b200 as paro  # noqa: E402
import synth  # noqa: E402

N, K, B = (int(v) for v in sys.argv[1:4])
dev = torch.device("cuda")
p = synth.make_problem(8, K, 1, seed=1)
s, th, pr = (torch.from_numpy(p[k]).to(dev) for k in ("s", "theta", "pairs"))
pk = paro.paro_pack((torch.randn(N, K, device=dev) * 0.02).half(), s, th, pr)
x = torch.randn(B, K, device=dev).half()
ws = torch.empty(paro.paro_linear_workspace(B, N, K), dtype=torch.uint8, device=dev)
for _ in range(3):
    y = paro.paro_linear(x, pk, workspace=ws)
torch.cuda.synchronize()
lib = ctypes.CDLL(paro.LIB_PATH)
buf = np.zeros(1024 * 4, dtype=np.uint64)
lib.paro_debug_pf_prof(buf.ctypes.data_as(ctypes.c_void_p), buf.size)
b = buf.reshape(1024, 4).astype(np.float64)
n = int((b[:, 3] > 0).sum())
b = b[:n]
tot = b[:, 3]
print(f"N={N} K={K} B={B}: {n} CTAs, MMA-thread cycles total median {np.median(tot):.0f} (max {tot.max():.0f})")
for i, name in enumerate(("acc_empty", "A stage", "x' stage")):
    print(f"  wait {name}: median {np.median(b[:, i] / tot) * 100:.1f}% of the CTA's cycles")
