"""Turn gpurun_out/prof (tools/profile_round.sh) into the committed summaries under profiles/<round>/
and profiles/traffic.json (read by bench.py for roofline.traffic).  argv: round_dir (e.g. profiles/r01)"""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "gpurun_out", "prof")
dst = os.path.join(ROOT, sys.argv[1])
os.makedirs(dst, exist_ok=True)

# 1. bench lines
shutil.copy(os.path.join(SRC, "bench.json"), os.path.join(dst, "bench.json"))
if os.path.exists(os.path.join(SRC, "bench_long.json")):
    shutil.copy(os.path.join(SRC, "bench_long.json"), os.path.join(dst, "bench_long.json"))

# 2. launch list of the bench under ncu (gpu__time_duration.sum): per-kernel shares
rows = [r for r in csv.reader(open(os.path.join(SRC, "launches.csv"))) if len(r) > 10]
hdr = rows[0]
ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if r[im] != "gpu__time_duration.sum":
        continue
    v = float(r[iv].replace(",", ""))
    unit = r[hdr.index("Metric Unit")]
    us = v / 1000.0 if unit in ("ns", "nsecond") else (v * 1000.0 if unit in ("ms", "msecond") else v)
    name = r[ik]
    if not name.startswith("void paro::") and not name.startswith("paro::"):
        name = name.split("(")[0][:80]  # torch helper kernels: short name
    a = agg[name]
    a[0] += 1
    a[1] += us
tot = sum(a[1] for a in agg.values())
with open(os.path.join(dst, "bench_launches_summary.csv"), "w") as f:
    f.write("# ncu launch list of `python bench.py --steps 3 --warmup 3 --no-cpu-baseline --load-s 0`\n")
    f.write("# gpu__time_duration.sum, --clock-control none; cold-cache serialised per-launch times: compare SHARES, not absolutes\n")
    f.write("kernel,launches,total_us,mean_us,share_of_all_launches\n")
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        f.write(f"\"{k}\",{n},{us:.1f},{us / n:.3f},{us / tot:.4f}\n")

# 3. ncu --set full of each decode group
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum.per_second", "dram__cycles_active.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__block_size",
        "launch__cluster_dim_x", "launch__registers_per_thread", "sm__cycles_active.avg", "sm__cycles_elapsed.avg",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tmem_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_uma.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
groups = {0: "q_proj+k_proj+v_proj (N=4096,1024,1024, K=4096), B=1", 1: "o_proj (N=4096, K=4096), B=1",
          2: "gate_proj+up_proj (N=14336 x2, K=4096), B=1", 3: "down_proj (N=4096, K=14336), B=1",
          4: "Qwen3-4B q/k/v (N=4096,1024,1024, K=2560), B=16, mma.sync engine",
          5: "Qwen3-4B q/k/v (N=4096,1024,1024, K=2560), B=16, tcgen05 engine",
          6: "LLaMA-3-70B down_proj (N=8192, K=28672), B=1, cross-cluster K split (7 slices, clusters of 2)",
          "prefill_q": "prefill GEMM q_proj (N=4096, K=4096), 2048 tokens (tcgen05)",
          "prefill_gate": "prefill GEMM gate_proj (N=14336, K=4096), 2048 tokens (tcgen05)",
          "prefill_transform": "prefill activation transform, dense tcgen05 form (2048 x 4096)"}
out = {"note": "ncu --set full --clock-control none, one launch each (tools/prof_multi.py, bs=1, rotation on); "
               "cold caches and ncu's replay: times are not bench values", "groups": {}}
traffic = 0.0
for i, name in groups.items():
    rep = os.path.join(SRC, f"group{i}.ncu-rep" if isinstance(i, int) else f"{i}.ncu-rep")
    if not os.path.exists(rep):
        continue
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    if len(r) < 3:
        continue
    h, u, v = r[0], r[1], r[2]
    m = {}
    stalls = []
    for a, b, c in zip(h, u, v):
        if a in keys:
            try:
                m[a] = {"value": float(c.replace(",", "")), "unit": b}
            except ValueError:
                m[a] = {"value": c, "unit": b}
        if a.startswith("smsp__pcsamp_warps_issue_stalled") and not a.endswith("not_issued"):
            try:
                stalls.append((int(float(c.replace(",", ""))), a.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    m["top_stalls"] = [s for _, s in sorted(stalls, reverse=True)[:6]]
    out["groups"][name] = m
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    if isinstance(i, int) and i < 4:  # the bench step's four launches
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            traffic += m[k]["value"] * scale.get(m[k]["unit"], 1)
json.dump(out, open(os.path.join(dst, "ncu_decode_groups.json"), "w"), indent=1)
json.dump({"traffic_per_step": round(traffic), "unit": "bytes",
           "source": f"{sys.argv[1]}/ncu_decode_groups.json: dram__bytes_read.sum + dram__bytes_write.sum of the "
                     "four decode launches of one bench step (ncu --set full)"},
          open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)
print("traffic per step", traffic, "launch share rows", len(agg))
