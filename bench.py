#!/usr/bin/env python
"""bench.py -- ParoQuant decode-linear benchmark on B200 (BASELINE.json metric:
"decode linear us & HBM GB/s (% of peak); rotation overhead vs plain W4A16").

One step = one pass of the runtime hot path (scale + 8 Givens
layers fused into the activation staging + group-wise INT4 dequant GEMV + epilogue)
over the seven linears of one LLaMA-3-8B decoder layer at bs=1 (BASELINE.json
configs[1]: q/k/v/o 4096x4096/1024, gate/up/down 4096x14336), random fp16 weights
packed with paro_pack (W4 g128, 8 Alg. A1 rotations) and random fp16 activations.
Steps cycle through a pool of layers whose packed weights exceed the 126 MB L2
(inputs larger than L2), so every step streams its weights from HBM.

value = algorithmic weight+param+activation bytes per step / device time per step
(GB/s, higher is better).  Multi-GPU (torchrun): every linear is sharded by output
channel across ranks and y is all-gathered with NCCL (strong scaling; value counts
the whole layer's bytes once).

--impl reference: the fp64 CPU oracle (oracle/) on a bounded sample of the same
workload, same metric (there is no reference implementation to install: the
reference is a paper).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "decode linear HBM GB/s (LLaMA-3-8B layer, bs=1, W4 g128, 8 Givens layers)"
WORKLOAD = "llama3-8b decode linears bs=1 (q,k,v,o,gate,up,down), W4 g128, L=8 rotations of <=64 pairs"
L2_BYTES = 126 * 1024 * 1024


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "_fallback": True}


def algorithmic_bytes(N, K, B=1, L=8, P=64):
    """W4A16 0.5195 B/weight + rotation params 6 B/pair + 4 B/channel s
    + activations 2BK in, 2BN out."""
    G = K // 128
    w = N * K // 2 + N * G * 2 + N * G // 2
    rot = G * L * P * 6 + 4 * K
    act = 2 * B * K + 2 * B * N
    return w + rot + act, w


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        import tempfile
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sms, mx, reasons = [], None, set()
        try:
            for line in open(self.path):
                f = [c.strip() for c in line.split(",")]
                if len(f) < 9:
                    continue
                try:
                    sms.append(float(f[1]))
                    mx = float(f[2])
                except ValueError:
                    continue
                names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
                for n, v in zip(names, f[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
        except Exception:
            pass
        if not sms:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sms), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sms)}


# ----------------------------------------------------------------------------- workload
def build_layer_pool(torch, paro, shapes, rank, world, n_layers, dev, seed=0):
    """Pack n_layers copies of the decoder layer's linears (this rank's row shard).
    Pairs/angles/scales are generated once per shape (speed does not depend on their
    values); the weights differ per layer."""
    G_cache = {}
    pool = []
    for li in range(n_layers):
        layer = []
        for name, (N, K) in shapes.items():
            if (N, K) not in G_cache:
                p = synth.make_problem(8, K, 1, seed=seed + N % 97)
                G_cache[(N, K)] = (torch.from_numpy(p["s"]).to(dev), torch.from_numpy(p["theta"]).to(dev),
                                   torch.from_numpy(p["pairs"]).to(dev))
            s, th, pr = G_cache[(N, K)]
            r0, r1 = paro.shard_rows(N, world, rank)
            g = torch.Generator(device=dev).manual_seed(seed * 1000 + li * 17 + N + K)
            W = (torch.randn((r1 - r0, K), generator=g, device=dev, dtype=torch.float32) * 0.02).to(torch.float16)
            packed = paro.paro_pack(W, s, th, pr)
            del W
            layer.append((name, N, K, packed))
        pool.append(layer)
    return pool


def clone_packed(paro, pk):
    """The same packed linear at new addresses (so a pool of clones is streamed from HBM)."""
    return paro.PackedLinear(pk.codes.clone(), pk.scales.clone(), pk.zeros.clone(), pk.rot_cs.clone(),
                             pk.rot_idx.clone(), pk.svec.clone(), pk.N, pk.K, pk.n_rot)


# the decode layer as chain stages: q/k/v share x, o reads the attention output (a separate
# input here), gate/up share x, down reads up's output (a real dependency inside the chain)
LAYER_STAGES = [["q_proj", "k_proj", "v_proj"], ["o_proj"], ["gate_proj", "up_proj"], ["down_proj"]]


def layer_chain(paro, layer, x_in, x_attn, ys):
    lin = {name: packed for name, N, K, packed in layer}
    return [paro.ChainStage(x_in, [lin[n] for n in LAYER_STAGES[0]], [ys[n] for n in LAYER_STAGES[0]]),
            paro.ChainStage(x_attn, [lin["o_proj"]], [ys["o_proj"]]),
            paro.ChainStage(x_in, [lin[n] for n in LAYER_STAGES[2]], [ys[n] for n in LAYER_STAGES[2]]),
            paro.ChainStage(ys["up_proj"], [lin["down_proj"]], [ys["down_proj"]])]


def pool_layers(world=1):
    """Layers in the weight pool: >= 4 x L2 of packed weights per rank (inputs larger than L2)."""
    wb = sum(algorithmic_bytes(N // world, K, 1)[1] for N, K in synth.LLAMA3_8B_DECODE.values())
    return min(64, max(2, int(np.ceil(4 * L2_BYTES / wb)))), wb


def bench_config(B, world=1):
    """The config block shared by both arms (pure arithmetic: the reference arm reports the same)."""
    n_layers, wb = pool_layers(world)
    return {"workload": WORKLOAD, "batch": B,
            "step": ("4 paro_linear_multi decode launches (q/k/v | o | gate/up | down reading up's y), "
                     "PDL-chained") if world == 1 else "7 paro_linear_allgather calls",
            "parallelism": f"N-shard x{world} + NCCL all-gather" if world > 1 else "single GPU",
            "l2": (f"inputs larger than L2: weight pool of {n_layers} layers x {wb / 1e6:.1f} MB/rank "
                   f"> 4 x 126 MB L2, cycled per step"),
            "bytes_per_step": sum(algorithmic_bytes(N, K, B)[0] for N, K in synth.LLAMA3_8B_DECODE.values())}


def run_paro(args):
    import torch
    import torch.distributed as dist

    import paper_2511_10645_b200 as paro

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)
    shapes = synth.LLAMA3_8B_DECODE
    B = args.batch
    comm = None
    if world > 1:
        from paper_2511_10645_b200 import dist as pd
        comm = pd.make_comm(rank, world)

    layer_bytes = sum(algorithmic_bytes(N, K, B)[0] for N, K in shapes.values())
    n_layers, _wb = pool_layers(world)
    pool = build_layer_pool(torch, paro, shapes, rank, world, n_layers, dev)
    g = torch.Generator(device=dev).manual_seed(123)
    # the step's inputs: x of the layer (q/k/v, gate/up) and the attention output (o); outputs are
    # views of one buffer (one copy per direction in e2e)
    x_all = torch.randn((2 * B * 4096,), generator=g, device=dev).to(torch.float16)
    x_in, x_attn = x_all[:B * 4096].view(B, 4096), x_all[B * 4096:].view(B, 4096)
    y_all = torch.empty((B * sum(N for N, _ in shapes.values()),), dtype=torch.float16, device=dev)
    ys, off = {}, 0
    for name, (N, K) in shapes.items():
        ys[name] = y_all[off:off + B * N].view(B, N)
        off += B * N
    ws = torch.empty(64 << 20, dtype=torch.uint8, device=dev)
    chains = [layer_chain(paro, layer, x_in, x_attn, ys) for layer in pool]
    chain_ws = paro.chain_workspace(B, chains[0])

    def run_step(li, flags, pdl=True):
        """One step: the layer's seven linears as four decode launches (q/k/v and gate/up share
        their input; down reads up's output), PDL-chained: each launch waits for its predecessor
        before reading x or writing y."""
        f = flags | (paro.PARO_LINEAR_PDL if pdl else 0)
        if world == 1:
            for st in chains[li % n_layers]:
                paro.paro_linear_multi(st.x, st.packed, y=st.y, flags=f, workspace=ws, stream=stream)
        else:
            layer = {name: (N, K, packed) for name, N, K, packed in pool[li % n_layers]}
            for grp in LAYER_STAGES:
                for name in grp:
                    N, K, packed = layer[name]
                    xin = ys["up_proj"] if name == "down_proj" else (x_attn if name == "o_proj" else x_in)
                    paro.paro_linear_allgather(xin, packed, comm, rank, world, y=ys[name], flags=f, workspace=ws,
                                               stream=stream)

    def run_step_chain(li, flags, pdl=True):
        """The same step as ONE persistent paro_linear_chain launch (grid barrier between stages)."""
        f = flags | (paro.PARO_LINEAR_PDL if pdl else 0)
        paro.paro_linear_chain(chains[li % n_layers], flags=f, workspace=chain_ws, stream=stream)

    def timed(step_fn, flags, steps, warmup):
        """Graph of `steps` consecutive steps (layers cycle through the pool); returns
        max-over-ranks ms per step measured with CUDA events on the launch stream."""
        gph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            for li in range(2):
                step_fn(li, flags)
            stream.synchronize()
            with torch.cuda.graph(gph, stream=stream):
                for li in range(steps):
                    step_fn(li, flags)
            for _ in range(max(1, warmup // max(steps, 1) + 1)):
                gph.replay()
            stream.synchronize()
            t_end = time.time() + args.load_s  # untimed load so the clock sampler sees the loaded state
            while time.time() < t_end:
                gph.replay()
                stream.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):  # CUDAGraph.replay() launches on the current stream
            e0.record(stream)
            gph.replay()
            e1.record(stream)
        e1.synchronize()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    # warm-up steps (untimed), then exactly K timed steps (in one graph replay)
    with ClockSampler(local) as clk:
        ms_step = timed(run_step, 0, args.steps, args.warmup)
    clocks = clk.summary()
    ms_norot = timed(run_step, paro.PARO_LINEAR_NO_ROTATION, args.steps, args.warmup)
    ms_chain = timed(run_step_chain, 0, args.steps, args.warmup) if world == 1 else None

    # cold single step: L2 flushed (a 2 x L2 buffer written) before each call, median of 7
    cold_us = None
    if world == 1:
        flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev)
        vals = []
        with torch.cuda.stream(stream):
            for i in range(8):
                flush.fill_(float(i))
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                run_step(i, 0, pdl=False)
                e1.record(stream)
                e1.synchronize()
                if i:
                    vals.append(e0.elapsed_time(e1) * 1e3)
        cold_us = round(statistics.median(vals), 2)
        del flush

    # per-linear timings, rotation on / off: each linear cycles through its own pool of clones
    # larger than 4 x L2 (inputs larger than L2), 100 calls per graph
    per_linear = {}
    if world == 1 and not args.no_extra:
        for name, (N, K) in shapes.items():
            base = [e for e in pool[0] if e[0] == name][0][3]
            nb = algorithmic_bytes(N, K, B)[1]
            n_cl = int(np.ceil(4 * L2_BYTES / nb))
            clones = [base] + [clone_packed(paro, base) for _ in range(n_cl - 1)]
            xin = x_attn if name == "o_proj" else (ys["up_proj"] if name == "down_proj" else x_in)
            res = {}
            for tag, fl in (("rot", 0), ("norot", paro.PARO_LINEAR_NO_ROTATION)):
                cnt = [0]

                def call():
                    pk = clones[cnt[0] % n_cl]
                    cnt[0] += 1
                    paro.paro_linear(xin, pk, y=ys[name], flags=fl | paro.PARO_LINEAR_PDL, workspace=ws, stream=stream)

                res[tag] = graph_time_us(torch, stream, call, max(100, n_cl))
            ab = algorithmic_bytes(N, K, B)[0]
            per_linear[name] = {"N": N, "K": K, "us": round(res["rot"], 3), "us_norot": round(res["norot"], 3),
                                "GBps": round(ab / res["rot"] / 1e3, 1), "pool_MB": round(n_cl * nb / 1e6),
                                "rot_overhead": round(res["rot"] / res["norot"] - 1.0, 4)}
            del clones
        torch.cuda.empty_cache()

    # end-to-end through the public API with host buffers (pinned), copies inside the timed region
    hx = x_all.cpu().pin_memory()
    hy = torch.empty(y_all.shape, dtype=torch.float16).pin_memory()
    h2d, d2h = hx.numel() * 2, hy.numel() * 2
    n_e2e = max(10, min(args.steps, 200))

    def e2e_step(li):
        # x in and y out over PCIe by the library's SM-driven copy (paro_copy), PDL-chained with the
        # decode launches: no DMA copy node breaks the programmatic-dependent chain
        with torch.cuda.stream(stream):
            paro.paro_copy(x_all, hx, flags=paro.PARO_LINEAR_PDL, stream=stream)
            run_step(li, 0, pdl=True)  # its x loads wait (PDL) for the copy before them
            paro.paro_copy(hy, y_all, flags=paro.PARO_LINEAR_PDL, stream=stream)

    for li in range(3):
        e2e_step(li)
    stream.synchronize()
    # the serving loop's form: each step (pinned-host x -> device, the decode chain, y -> pinned
    # host) captured once in a CUDA graph and replayed; the copies run every step
    per_graph = n_layers
    gph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        with torch.cuda.graph(gph, stream=stream):
            for li in range(per_graph):
                e2e_step(li)
        gph.replay()
        stream.synchronize()
    reps = max(1, n_e2e // per_graph)
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(reps):
            gph.replay()
        e1.record(stream)
    e1.synchronize()
    ms_e2e = e0.elapsed_time(e1) / (reps * per_graph)
    if world > 1:
        t = torch.tensor([ms_e2e], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t.item())
    del gph
    e2e = {"value": round(layer_bytes / (ms_e2e * 1e-3) / 1e9, 2), "unit": "GB/s", "ms_per_step": round(ms_e2e, 4),
           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
           "api": ("paper_2511_10645_b200.paro_linear_multi (4 decode launches per step)" if world == 1 else
                   "paper_2511_10645_b200.paro_linear_allgather per linear") +
                  " with the pinned-host x -> device and y -> host copies of every step (paro_copy: SM-driven "
                  "PCIe copies, PDL-chained with the decode launches), each step captured in a CUDA graph and "
                  "replayed"}

    # prefill (SURVEY.md 8(d) "also prefill TFLOPS"): the same packed linears at 2048 tokens
    # through paro_linear's tcgen05 path (transform pre-stage + GEMM), one CUDA graph per linear
    prefill = None
    if world == 1 and not args.no_prefill:
        prefill = measure_prefill(torch, paro, dev, stream, pool[0], g)

    extra = {}
    if world == 1 and not args.no_extra:
        extra["c1"] = measure_c1(torch, paro, dev, stream)
        extra["transform_vs_fwht"] = measure_transform_vs_fwht(torch, paro, dev, stream)
        extra["c3_qwen3_4b_stack"] = measure_qwen_stack(torch, paro, dev, stream, (1, 4, 16))
    del pool, chains
    torch.cuda.empty_cache()
    if not args.no_extra:
        # configs[4]: the LLaMA-3-70B MLP, N-sharded over the ranks of this run (1 GPU: the whole
        # layer), GEMV and all-gather reported separately
        extra["c5_llama3_70b_mlp"] = measure_70b_mlp(torch, paro, dev, stream, comm, rank, world)

    if comm is not None:
        torch.cuda.synchronize()
        paro.paro_comm_destroy(comm)
    if world > 1:
        dist.barrier()
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peaks = load_peaks()
    gbps = layer_bytes / (ms_step * 1e-3) / 1e9
    peak = float(peaks.get("hbm_gbs", 6650.0))
    out = {
        "metric": METRIC, "value": round(gbps, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 5), "us_per_step": round(ms_step * 1e3, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f16 act / int4 weight / f32 acc",
        "rotation_overhead": round(ms_step / ms_norot - 1.0, 4), "us_per_step_norot": round(ms_norot * 1e3, 3),
        "frac_of_8TBps": round(gbps / 8000.0, 4),
        "us_per_step_chain": None if ms_chain is None else round(ms_chain * 1e3, 3),
        "cold_step_us": cold_us,
        "data": "synthetic (random fp16 W ~ N(0,0.02^2) packed W4 g128 with Alg. A1 pairs, random theta/s; x ~ N(0,1))",
        "config": bench_config(B, world),
        "roofline": {"bound": "hbm", "achieved": round(gbps, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(gbps / peak, 4), "traffic": None,
                     "kernel": "paro_gemv1_b1_kernel (the step's 4 decode launches)",
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, burst)" if not peaks.get("_fallback")
                     else "fallback 6.65 TB/s",
                     "achieved_def": "algorithmic bytes per step (SURVEY.md 8(d): 0.5195 B/weight + 6 B/pair + 4 B/ch "
                                     "s + 2BK + 2BN) / device time per step"},
        "clocks": clocks, "e2e": e2e,
        "gpu_launches": (4 if world == 1 else 14) * args.steps,
        "gpu_launches_note": ("4 paro_gemv1_b1_kernel launches per step (q/k/v and gate/up fused by shared input)"
                              if world == 1 else "7 paro_gemv1_b1_kernel + 7 ncclAllGather launches per step"),
        "per_linear": per_linear, "prefill": prefill, **extra,
    }
    if world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args)
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        out["roofline"]["traffic"] = prof.get("traffic_per_step")
        out["roofline"]["traffic_src"] = prof.get("source")
    except Exception:
        pass
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def graph_time_us(torch, stream, fn, reps):
    """Device time per call of fn() captured reps times in one CUDA graph (CUDA events)."""
    with torch.cuda.stream(stream):
        fn()
        fn()
        stream.synchronize()
        gph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gph, stream=stream):
            for _ in range(reps):
                fn()
        gph.replay()
        stream.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        gph.replay()
        e1.record(stream)
        e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def measure_transform_vs_fwht(torch, paro, dev, stream, tokens=(1, 2048)):
    """SURVEY.md 8(f) NEXT #2, the paper's kernel experiment (fig:kernel-speedup):
    the standalone scaled pairwise rotation (paro_transform_activations: s, then 8 rotations of
    <= 64 pairs per 128-channel group) vs the fast Walsh-Hadamard transform over all n channels
    (paro_fwht, randomised: signs, butterfly, 1/sqrt(n)), same fp16 activations, fp16 outputs,
    device time per call (graph of repeated calls)."""
    out = {}
    for n in (256, 512, 1024, 2048, 4096, 8192, 16384):
        p = synth.make_problem(32, n, 1, seed=n)
        t = {k: torch.from_numpy(p[k]).to(dev) for k in ("W", "s", "theta", "pairs")}
        packed = paro.paro_pack(t["W"], t["s"], t["theta"], t["pairs"])
        signs = torch.from_numpy(np.random.default_rng(n).choice([-1.0, 1.0], size=n).astype(np.float32)).to(dev)
        row = {}
        for T in tokens:
            x = torch.randn((T, n), device=dev).to(torch.float16)
            yr = torch.empty((T, n), dtype=torch.float16, device=dev)
            yf = torch.empty((T, n), dtype=torch.float16, device=dev)
            reps = 50 if T <= 16 else 20
            ur = graph_time_us(torch, stream, lambda: paro.paro_transform_activations(x, packed, out=yr, stream=stream),
                               reps)
            uf = graph_time_us(torch, stream, lambda: paro.paro_fwht(x, signs, 1.0 / np.sqrt(n), out=yf, stream=stream),
                               reps)
            row[f"T{T}"] = {"rotation_us": round(ur, 3), "fwht_us": round(uf, 3), "speedup": round(uf / ur, 3)}
            if T >= 64:  # the same transform as a dense per-group contraction (the prefill path's form)
                yd = torch.empty((T, n), dtype=torch.float16, device=dev)
                wsd = torch.empty(paro._lib.paro_transform_dense_workspace(n), dtype=torch.uint8, device=dev)
                ud = graph_time_us(torch, stream, lambda: paro.paro_transform_activations_dense(
                    x, packed, out=yd, workspace=wsd, stream=stream), reps)
                row[f"T{T}"].update({"dense_rotation_us": round(ud, 3), "speedup_dense": round(uf / ud, 3)})
        out[str(n)] = row
    return out


def measure_c1(torch, paro, dev, stream):
    """configs[0]: one K = N = 256 linear, bs=1 (launch-latency bound: report us)."""
    p = synth.make_problem(256, 256, 1, seed=7)
    t = {k: torch.from_numpy(p[k]).to(dev) for k in ("W", "s", "theta", "pairs", "x")}
    packed = paro.paro_pack(t["W"], t["s"], t["theta"], t["pairs"])
    y = torch.empty((1, 256), dtype=torch.float16, device=dev)
    res = {}
    for tag, fl in (("rot", 0), ("norot", paro.PARO_LINEAR_NO_ROTATION), ("rot_pdl", paro.PARO_LINEAR_PDL)):
        res[tag] = graph_time_us(torch, stream, lambda: paro.paro_linear(t["x"], packed, y=y, flags=fl, stream=stream),
                                 200)
    return {"us": round(res["rot"], 3), "us_norot": round(res["norot"], 3),
            "rot_overhead": round(res["rot"] / res["norot"] - 1.0, 4), "us_pdl": round(res["rot_pdl"], 3),
            "def": "device time per paro_linear call, 200 calls in one CUDA graph (weights L2-resident); us_pdl: "
                   "the calls PDL-chained (each call's prologue overlaps the previous call's tail)"}


def measure_prefill(torch, paro, dev, stream, layer, g):
    """The layer's linears at 2048 tokens through paro_linear's tcgen05 path (transform
    pre-stage + GEMM), one CUDA graph per linear; TFLOP/s = 2 B N K / device time."""
    Bp = 2048
    tot_flop, tot_us, per = 0.0, 0.0, {}
    with torch.cuda.stream(stream):
        for name, N, K, packed in layer:
            xp = torch.randn((Bp, K), generator=g, device=dev).to(torch.float16)
            yp = torch.empty((Bp, N), dtype=torch.float16, device=dev)
            wsp = torch.empty(max(1, paro.paro_linear_workspace(Bp, N, K)), dtype=torch.uint8, device=dev)
            us = graph_time_us(torch, stream, lambda: paro.paro_linear(xp, packed, y=yp, workspace=wsp, stream=stream),
                               10)
            fl = 2.0 * Bp * N * K
            tot_flop += fl
            tot_us += us
            per[name] = {"us": round(us, 2), "TFLOPs": round(fl / us / 1e6, 1)}
            del xp, yp, wsp
    pk = load_peaks()
    tpeak = float(pk.get("bf16_tflops", 1649.0))
    speak = pk.get("bf16_tflops_sustained")
    tf = tot_flop / tot_us / 1e6
    return {"tokens": Bp, "TFLOPs": round(tf, 1), "us_per_layer": round(tot_us, 1),
            "peak_TFLOPs": tpeak, "frac": round(tf / tpeak, 4),
            "peak_sustained_TFLOPs": speak, "frac_sustained": round(tf / float(speak), 4) if speak else None,
            "per_linear": per,
            "def": "2*B*N*K flop per linear / device time of transform pre-stage + tcgen05 GEMM; peak: "
                   "MEASURED_PEAKS.json bf16 burst (fp16 dense = bf16 rate); the layer is ~0.9 ms of back-to-back "
                   "GEMMs that run power-limited, so the sustained figure is the matching denominator"}


def measure_qwen_stack(torch, paro, dev, stream, batches):
    """configs[2]: the Qwen3-4B decode stack (36 layers x 7 linears, each with its own
    transform), every layer 4 decode launches (q/k/v | o | gate/up | down reading up's y): 144
    PDL-chained launches per step (also timed as 9 persistent chain launches); 1.9 GB of packed
    weights, so every step streams from HBM.  Bytes per step include the B-token activations
    (SURVEY.md 8(d))."""
    shapes = synth.QWEN3_4B_LAYER
    pool = build_layer_pool(torch, paro, shapes, 0, 1, synth.QWEN3_4B_LAYERS, dev, seed=11)
    out = {"layers": synth.QWEN3_4B_LAYERS}
    for B in batches:
        step_bytes = sum(algorithmic_bytes(N, K, B)[0] for N, K in shapes.values()) * synth.QWEN3_4B_LAYERS
        g = torch.Generator(device=dev).manual_seed(5 + B)
        x_in = torch.randn((B, 2560), generator=g, device=dev).to(torch.float16)
        x_attn = torch.randn((B, 4096), generator=g, device=dev).to(torch.float16)
        ys = {n: torch.empty((B, N), dtype=torch.float16, device=dev) for n, (N, K) in shapes.items()}
        stages = []
        for layer in pool:
            stages += layer_chain(paro, layer, x_in, x_attn, ys)
        ws = torch.empty(64 << 20, dtype=torch.uint8, device=dev)

        def step(fl):
            for st in stages:  # 144 PDL-chained decode launches
                paro.paro_linear_multi(st.x, st.packed, y=st.y, flags=fl | paro.PARO_LINEAR_PDL, workspace=ws,
                                       stream=stream)

        res = {}
        for tag, fl in (("rot", 0), ("norot", paro.PARO_LINEAR_NO_ROTATION)):
            res[tag] = graph_time_us(torch, stream, lambda: step(fl), 3)
        try:  # the same stack as persistent chains (16 stages per launch)
            cws = paro.chain_workspace(B, stages)
            res["chain"] = graph_time_us(torch, stream, lambda: paro.paro_linear_chain(
                stages, flags=paro.PARO_LINEAR_PDL, workspace=cws, stream=stream), 3)
        except Exception:  # noqa: BLE001  (a chain plan may not fit shared memory at 16 tokens)
            res["chain"] = None
        out[f"bs{B}"] = {"us_per_step": round(res["rot"], 1), "GBps": round(step_bytes / res["rot"] / 1e3, 1),
                         "bytes_per_step": int(step_bytes), "rot_overhead": round(res["rot"] / res["norot"] - 1.0, 4),
                         "us_per_step_chain": None if res["chain"] is None else round(res["chain"], 1)}
        del stages, ws
    del pool
    torch.cuda.empty_cache()
    return out


def measure_70b_mlp(torch, paro, dev, stream, comm, rank, world):
    """configs[4]: the LLaMA-3-70B MLP linears (gate/up 8192 -> 28672, down 28672 -> 8192) at
    bs=1, rows sharded over the `world` ranks of this run; two layer copies
    alternate, so every call streams from HBM.  Reported per rank: the shard GEMV alone, the
    GEMV + NCCL all-gather (paro_linear_allgather; world 1: the plain GEMV), and their difference
    as the all-gather cost; max over ranks."""
    import torch.distributed as dist
    shapes = synth.LLAMA3_70B_MLP
    pool = build_layer_pool(torch, paro, shapes, rank, world, 2, dev, seed=23)
    x = torch.randn((1, 8192), device=dev).to(torch.float16)
    ys = {n: torch.zeros((1, N), dtype=torch.float16, device=dev) for n, (N, K) in shapes.items()}
    ysh = {n: torch.zeros((1, N // world), dtype=torch.float16, device=dev) for n, (N, K) in shapes.items()}
    ws = torch.empty(16 << 20, dtype=torch.uint8, device=dev)
    out = {"world": world}
    tot = {"gemv_us": 0.0, "total_us": 0.0, "p2p_total_us": 0.0}
    from paper_2511_10645_b200 import dist as pd
    p2p = {}
    p2p_ok = 1
    try:  # CUDA IPC peer mappings for the NVLink-native exchange (every rank must succeed)
        for name, (N, K) in shapes.items():
            buf, ptrs, opened = pd.make_p2p(rank, world, N, torch.float16, device=dev) if world > 1 else \
                (paro.p2p_buffer(N, 1, torch.float16, device=dev), None, [])
            p2p[name] = (buf, ptrs if ptrs is not None else [buf.data_ptr()], opened)
    except Exception as ex:  # noqa: BLE001 -- reported, and the P2P timing is skipped on every rank
        p2p_ok = 0
        print(f"[bench] rank {rank}: P2P exchange setup failed ({ex}); skipping the p2p timing", file=sys.stderr)
    if world > 1:
        t = torch.tensor([p2p_ok], device=dev, dtype=torch.int32)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        p2p_ok = int(t.item())
    for name, (N, K) in shapes.items():
        xin = ys["up_proj"] if name == "down_proj" else x
        res = {}
        for tag in ("gemv", "total", "norot", "p2p"):
            if tag == "p2p" and not p2p_ok:
                res[tag] = float("nan")
                continue
            cnt = [0]

            def call():
                pk = [e for e in pool[cnt[0] % 2] if e[0] == name][0][3]
                cnt[0] += 1
                if tag == "total" and world > 1:
                    paro.paro_linear_allgather(xin, pk, comm, rank, world, y=ys[name], flags=paro.PARO_LINEAR_PDL,
                                               workspace=ws, stream=stream)
                elif tag == "p2p":  # the NVLink-native exchange (GEMV epilogue peer stores + flags)
                    buf, ptrs, _ = p2p[name]
                    paro.paro_linear_allgather_p2p(xin, pk, ptrs, rank, world, buf, flags=paro.PARO_LINEAR_PDL,
                                                   stream=stream)
                else:
                    fl = paro.PARO_LINEAR_NO_ROTATION if tag == "norot" else 0
                    paro.paro_linear(xin, pk, y=ysh[name], flags=fl | paro.PARO_LINEAR_PDL, workspace=ws,
                                     stream=stream)

            us = graph_time_us(torch, stream, call, 20)
            if world > 1:
                t = torch.tensor([us], device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                us = float(t.item())
            res[tag] = us
        nbytes = algorithmic_bytes(N // world, K, 1)[0]
        out[name] = {"gemv_us": round(res["gemv"], 2), "allgather_us": round(res["total"] - res["gemv"], 2),
                     "total_us": round(res["total"], 2),
                     "p2p_total_us": round(res["p2p"], 2) if p2p_ok else None,
                     "GBps_per_gpu": round(nbytes / res["gemv"] / 1e3, 1),
                     "rot_overhead": round(res["gemv"] / res["norot"] - 1.0, 4)}
        tot["gemv_us"] += res["gemv"]
        tot["total_us"] += res["total"]
        tot["p2p_total_us"] += res["p2p"]
    all_bytes = sum(algorithmic_bytes(N, K, 1)[0] for N, K in shapes.values())
    out["mlp"] = {"gemv_us": round(tot["gemv_us"], 2), "allgather_us": round(tot["total_us"] - tot["gemv_us"], 2),
                  "total_us": round(tot["total_us"], 2),
                  "p2p_total_us": round(tot["p2p_total_us"], 2) if p2p_ok else None,
                  "aggregate_GBps": round(all_bytes / tot["total_us"] / 1e3, 1),
                  "def": "one call per linear (gate, up, down reading up's y), each timed alone in a graph of 20"}
    for buf, ptrs, opened in p2p.values():
        for q in opened:
            paro.paro_ipc_close_handle(q)
    del pool, p2p
    torch.cuda.empty_cache()
    return out


# ----------------------------------------------------------------------------- the oracle as baseline
def oracle_sample(frac_rows=0.125, seed=0):
    """A bounded sample of one step for the fp64 oracle: every linear of the layer, a
    fraction of its output rows (rows are independent in the fold, the RTN and the dot).
    The oracle pack (offline) is done here, untimed."""
    import oracle as O
    items = []
    for name, (N, K) in synth.LLAMA3_8B_DECODE.items():
        n = max(1, int(N * frac_rows))
        p = synth.make_problem(n, K, 1, seed=seed + N % 97, outliers=False)
        pk = O.oracle_pack(p["W"], p["s"], p["theta"], p["pairs"])
        items.append((p, pk, algorithmic_bytes(n, K, 1)[0]))
    return items


def oracle_time(items):
    """Run oracle_linear (scale + rotations + fp64 dequant-dot) over the sample; (bytes, s)."""
    import oracle as O
    tb, tt = 0, 0.0
    for p, pk, b in items:
        t0 = time.perf_counter()
        O.oracle_linear(p["x"], pk, p["s"], p["theta"], p["pairs"])
        tt += time.perf_counter() - t0
        tb += b
    return tb, tt


def cpu_baseline(args):
    from threadpoolctl import threadpool_limits
    items = oracle_sample(0.125)
    with threadpool_limits(limits=1):
        oracle_time(items)  # warm
        b, t = oracle_time(items)
    # also the oracle with every host core the process may use (BLAS threads)
    n_all = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    with threadpool_limits(limits=n_all):
        oracle_time(items)
        b2, t2 = oracle_time(items)
    return {"value": round(b / t / 1e9, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
            "all_cores": {"value": round(b2 / t2 / 1e9, 4), "cores": n_all},
            "sample": "oracle_linear (fp64 numpy) on 1/8 of the output rows of each of the 7 LLaMA-3-8B linears, "
                      "bs=1, BLAS limited to 1 thread (all_cores: to every core of the affinity mask); "
                      "oracle pack (offline) untimed"}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from threadpoolctl import threadpool_limits
    frac = 1.0 / 64
    items = oracle_sample(frac)
    with threadpool_limits(limits=1):
        for _ in range(args.warmup):
            oracle_time(items)
        tb, tt = 0, 0.0
        for i in range(args.steps):
            b, t = oracle_time(items)
            tb += b
            tt += t
    v = tb / tt / 1e9
    ms = tt / args.steps * 1e3
    sample = ("oracle_linear (fp64 numpy, 1 thread) on 1/64 of the output rows of each of the 7 LLaMA-3-8B "
              "linears per step, bs=1; oracle pack (offline) done once, untimed")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(1, world),
        "cpu_baseline": {"value": round(v, 4), "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": round(v, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--impl", default="paro", choices=["paro", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--load-s", type=float, default=1.0)
    ap.add_argument("--no-prefill", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the C1 / Qwen3-4B stack lines")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_paro(args)


if __name__ == "__main__":
    main()
