#!/bin/bash
# SM clock / power / throttle reasons sampled while a prefill GEMM runs back to back (evidence for
# the power-limited prefill GEMM).  -> stdout
rm -f /tmp/go
python - <<'PY' &
import sys, time, os
sys.path.insert(0, ".")
import torch, synth, paper_2511_10645_b200 as paro
dev = torch.device("cuda")
N, K, B = 14336, 4096, 2048
p = synth.make_problem(8, K, 1, seed=1)
s, th, pr = (torch.from_numpy(p[k]).to(dev) for k in ("s", "theta", "pairs"))
pk = paro.paro_pack((torch.randn(N, K, device=dev) * 0.02).half(), s, th, pr)
x = torch.randn(B, K, device=dev).half()
y = torch.empty(B, N, device=dev).half()
ws = torch.empty(paro.paro_linear_workspace(B, N, K), dtype=torch.uint8, device=dev)
for _ in range(5):
    paro.paro_linear(x, pk, y=y, workspace=ws, flags=paro.PARO_LINEAR_PDL)
torch.cuda.synchronize()
open("/tmp/go", "w").close()
t0 = time.time()
n = 0
while time.time() - t0 < 8:
    for _ in range(100):
        paro.paro_linear(x, pk, y=y, workspace=ws, flags=paro.PARO_LINEAR_PDL)
    torch.cuda.synchronize()
    n += 100
print(f"prefill gate_proj: {n} calls in {time.time() - t0:.1f} s = {(time.time() - t0) / n * 1e6:.1f} us per call", flush=True)
PY
PY_PID=$!
while [ ! -f /tmp/go ]; do sleep 0.1; done
sleep 1
for i in $(seq 1 24); do nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv,noheader; sleep 0.25; done > /tmp/clk.txt
wait $PY_PID
echo "samples during the run (SM clock, power, throttle-reason bits):"
sort /tmp/clk.txt | uniq -c | sort -rn | head -10
