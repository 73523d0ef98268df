"""Per-CTA timeline of the LLaMA-3-8B decode step (bs=1, four PDL-chained paro_linear_multi
launches of paro_gemv1_b1_kernel), as in bench.py.  Needs the library built with
PARO_NVCC_EXTRA=-DPARO_TIMELINE=1 (tools/tl_b1.sh).  Events per (CTA, launch):
0 start (setup done), 1 PDL wait returned (warp 0), 2 x loaded + scaled (warp 0), 3 transform
done (CTA), 4 first ring stage landed, 5 tiles done, 6 cluster partials in, 7 y stored,
8 producer issued its last stage, 9 producer released behind the x loads, 10 producer passed the
parameter barrier.  Events are clock64 within the CTA, placed on the %globaltimer of event 0."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2511_10645_b200 as paro  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda")
shapes = synth.LLAMA3_8B_DECODE
n_layers = 5
pool = bench.build_layer_pool(torch, paro, shapes, 0, 1, n_layers, dev)
x_in = torch.randn(1, 4096, device=dev).half()
x_attn = torch.randn(1, 4096, device=dev).half()
ys = {n: torch.empty(1, N, device=dev, dtype=torch.half) for n, (N, K) in shapes.items()}
chains = [bench.layer_chain(paro, layer, x_in, x_attn, ys) for layer in pool]
st = torch.cuda.Stream()
reps = 4  # 4 steps x 4 launches = the 16 timeline slots
lib = ctypes.CDLL(paro.LIB_PATH)


def step(li):
    for s in chains[li % n_layers]:
        paro.paro_linear_multi(s.x, s.packed, y=s.y, flags=paro.PARO_LINEAR_PDL, stream=st)


with torch.cuda.stream(st):
    step(0)
    st.synchronize()
    lib.paro_debug_b1_seq_reset()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for i in range(reps):
            step(i)
    for _ in range(3):
        g.replay()
    st.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    g.replay()
    e1.record(st)
    e1.synchronize()
print(f"{e0.elapsed_time(e1) / reps * 1e3:.2f} us per step", flush=True)
buf = np.zeros(1024 * 16 * 12, dtype=np.uint64)
lib.paro_debug_timeline_b1(buf.ctypes.data_as(ctypes.c_void_p), buf.size)
raw = buf.reshape(1024, 16, 12).astype(np.int64)
MHZ = float(os.environ.get("SM_MHZ", "1965"))
tl = np.zeros((1024, 16, 11), dtype=np.float64)
for e in range(11):
    ok = (raw[:, :, e] > 0) & (raw[:, :, 11] > 0)
    tl[:, :, e] = np.where(ok, raw[:, :, 11] + (raw[:, :, e] - raw[:, :, 0]) * 1e3 / MHZ, 0)
names = ["start", "pdl", "x", "xform", "st0", "tiles", "recv", "stored", "prod_end", "prod_rel", "prod_bar3"]
t0 = None
for s in range(8, 16):
    v0 = tl[:, s, 0]
    n = int((v0 > 0).sum())
    if t0 is None:
        t0 = v0[v0 > 0].min()
    row = []
    for e in range(len(names)):
        v = tl[:n, s, e]
        v = v[v > 0]
        if len(v) == 0:
            row.append(f"{names[e]}=-")
            continue
        row.append(f"{names[e]}={(np.median(v) - t0) / 1e3:.2f}[{(v.min() - t0) / 1e3:.2f},{(v.max() - t0) / 1e3:.2f}]")
    print(f"launch {s - 8} ({n} CTAs): " + " ".join(row), flush=True)
print("intra-CTA: median cycles after event 0 (start), per launch of the last step", flush=True)
for s in range(12, 16):
    n = int((raw[:, s, 0] > 0).sum())
    row = []
    for e in range(1, 11):
        v = raw[:n, s, e]
        ok = v > 0
        d = (v[ok] - raw[:n, s, 0][ok])
        row.append(f"{names[e]}={int(np.median(d)) if len(d) else -1}")
    print(f"launch {s - 12}: " + " ".join(row), flush=True)
np.save(os.path.join(ROOT, "gpurun_out", "tl", "b1_raw.npy"), raw)
st = np.zeros(4 * 1024 * 64 * 3, dtype=np.uint64)
lib.paro_debug_timeline_b1_st(st.ctypes.data_as(ctypes.c_void_p), st.size)
st = st.reshape(4, 1024, 64, 3).astype(np.int64)
for li, s in ((0, 12), (1, 13), (2, 14), (3, 15)):
    n = int((raw[:, s, 0] > 0).sum())
    c0 = raw[:n, s, 0][:, None]
    iss, rdy, don = (st[li, :n, :, e] for e in range(3))
    nst = int((rdy[0] > 0).sum())
    print(f"launch {s - 12} per stage (median cycles after start over CTAs; CTA 0 has {nst} stages): "
          "issued / data-ready (warp 0) / consumed (warp 0)", flush=True)
    for k in range(min(nst, 20)):
        def med(a):
            v = a[:, k]
            ok = v > 0
            return int(np.median(v[ok] - c0[ok, 0])) if ok.any() else -1
        print(f"  stage {k}: {med(iss)} / {med(rdy)} / {med(don)}", flush=True)
tt = np.zeros(1024 * 16 * 4, dtype=np.uint64)
if hasattr(lib, "paro_debug_timeline_b1_tile"):
    lib.paro_debug_timeline_b1_tile(tt.ctypes.data_as(ctypes.c_void_p), tt.size)
    tt = tt.reshape(1024, 16, 4).astype(np.int64)
    s = 13
    n = int((raw[:, s, 0] > 0).sum())
    st0 = st[1, :n, 0, 1]  # stage 0 data-ready (thread 0) of launch slot 13
    print("o_proj per-warp tile completion (median cycles after stage-0 data-ready, over CTAs):", flush=True)
    for w in (0, 4, 8, 15):
        row = []
        for k in range(2):
            v = tt[:n, w, k]
            ok = (v > 0) & (st0 > 0)
            row.append(int(np.median(v[ok] - st0[ok])) if ok.any() else -1)
        print(f"  warp {w}: tile 0 done +{row[0]}, tile 1 done +{row[1]}", flush=True)
