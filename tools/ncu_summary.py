"""Summarise an ncu report: top stall reasons, key metrics, SASS opcode mix.  argv: report.ncu-rep"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, u, v = r[0], r[1], r[2]
st = []
keys = ("gpu__time_duration.sum", "sm__cycles_active.avg", "sm__cycles_elapsed.avg", "smsp__inst_executed.sum",
        "launch__grid_size", "launch__block_size", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__warps_active.avg.per_cycle_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "launch__registers_per_thread", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active")
for a, b, c in zip(h, u, v):
    if a.startswith("smsp__pcsamp_warps_issue_stalled") and not a.endswith("not_issued"):
        try:
            x = float(c.replace(",", ""))
            if x > 0:
                st.append((int(x), a.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
    if a in keys:
        print(f"  {a} [{b}] {c}")
print("stalls:", sorted(st, reverse=True)[:12])
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(src.splitlines()))
hh = rows[1]
ia, isrc, ist = hh.index("Instructions Executed"), hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)")
tot = 0
byop = collections.Counter()
stl = collections.Counter()
for x in rows[2:]:
    try:
        n = int(x[ia])
    except (ValueError, IndexError):
        continue
    parts = x[isrc].split()
    if not parts:
        continue
    op = parts[1] if parts[0].startswith("@") and len(parts) > 1 else parts[0]
    op = op.split(".")[0]
    byop[op] += n
    tot += n
    stl[op] += int(x[ist] or 0)
print("inst total", tot)
for op, n in byop.most_common(22):
    print(f"  {op:10s} {n:9d} {n / tot * 100:5.1f}%  stall-samples {stl[op]}")
