"""Per-CTA event timeline of one decode launch (internal debug flag 0x100; needs a library built with
PARO_NVCC_EXTRA=-DPARO_ENABLE_DEBUG=1).
argv: N K (rot|norot) [graph_prev=1]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_10645_b200 as paro  # noqa: E402
import synth  # noqa: E402

N, K, mode = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
nlin = int(sys.argv[4]) if len(sys.argv) > 4 else 1
dev = torch.device("cuda")
p = synth.make_problem(8, K, 1, seed=1)
s, th, pr = (torch.from_numpy(p[k]).to(dev) for k in ("s", "theta", "pairs"))
pks = [[paro.paro_pack((torch.randn(N, K, device=dev) * 0.02).half(), s, th, pr) for _ in range(nlin)]
       for _ in range(2)]
Bt = int(os.environ.get("TL_B", "1"))
x = torch.randn(Bt, K, device=dev).half()
ys = [torch.empty(Bt, N, device=dev, dtype=torch.half) for _ in range(nlin)]
fl = paro.PARO_LINEAR_NO_ROTATION if mode == "norot" else 0
lib = paro._lib
lib.paro_debug_read_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int]
for it in range(3):
    paro.paro_linear_multi(x, pks[0], y=ys, flags=fl)
    torch.cuda.synchronize()
    paro.paro_linear_multi(x, pks[1], y=ys, flags=fl | 0x100)
    torch.cuda.synchronize()
buf = np.zeros(1024 * 12, dtype=np.uint64)
lib.paro_debug_read_timeline(buf.ctypes.data, buf.size)
t = buf.reshape(1024, 12).astype(np.int64)
live = t[:, 0] > 0
t = t[live]
t0 = t[:, 0].min()
rel = (t - t0) / 1000.0
names = ["start", "x_arrived", "transform_done", "stage0_ready", "loop_done", "end", "w0_layers_done", "w0_item_out", "w0_layers_start", "stage0_landed(producer)", "reach_stage0_wait", "last_stage_landed"]
print(f"{mode} N={N}x{nlin} K={K}: {live.sum()} CTAs; us relative to first CTA start")
for i, n in enumerate(names):
    col = rel[:, i]
    print(f"  {n:15s} min {col.min():7.2f}  median {np.median(col):7.2f}  max {col.max():7.2f}")

lib.paro_debug_read_prof.argtypes = [ctypes.c_void_p, ctypes.c_int]
pb = np.zeros(1024 * 16 * 8, dtype=np.uint64)
lib.paro_debug_read_prof(pb.ctypes.data, pb.size)
pb = pb.reshape(1024, 16, 8)[: live.sum()].astype(np.int64)
wait, work = pb[:, :, 0], pb[:, :, 1]
act = (wait + work) > 0
print(f"  phase-2 per warp (cycles): wait median {np.median(wait[act]):.0f} max {wait[act].max()}  work median {np.median(work[act]):.0f} max {work[act].max()}")
print(f"  stages/CTA median {np.median(pb[:, 0, 2]):.0f}  tiles/CTA median {np.median(pb[:, 0, 3]):.0f}  work cycles per tile-per-warp {np.median(work[act]) / max(1, np.median(pb[:, 0, 3]) / max(1, act.sum(1).max())):.0f}")
w0 = pb[:, 0, :]
print(f"  phase-1 warp 0 (cycles): params+x+scale median {np.median(w0[:, 4]):.0f}  rotations {np.median(w0[:, 5]):.0f}  output {np.median(w0[:, 6]):.0f}  x'-wait {np.median(w0[:, 7]):.0f}")
