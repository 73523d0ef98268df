#!/bin/bash
# Same-box A/B of a compile-time switch: bash tools/ab_flag.sh "<nvcc -D flags A>" "<flags B>" [rounds]
# Rebuilds libparo.so per variant and prints the bench step, Qwen3-4B bs1 stack and C5 per variant.
A=$1; B=$2; N=${3:-2}
for r in $(seq $N); do
  for v in "$A" "$B"; do
    PARO_NVCC_EXTRA="$v" python -c "from importlib import util; import sys; sys.path.insert(0,'.'); spec=util.spec_from_file_location('b','paper_2511_10645_b200/_build.py'); m=util.module_from_spec(spec); spec.loader.exec_module(m); m.build(force=True)" > /dev/null 2>&1 || { echo "build failed: $v"; exit 1; }
    echo "== [$v]"
    python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
c5=d.get('c5_llama3_70b_mlp') or {}
print('step', d['us_per_step'], 'norot', d.get('us_per_step_norot'), 'c1', d['c1']['us'], 'qwen bs1', d['c3_qwen3_4b_stack']['bs1']['us_per_step'],
      'bs4', d['c3_qwen3_4b_stack']['bs4']['us_per_step'], '70B gate/down', (c5.get('gate_proj') or {}).get('gemv_us'), (c5.get('down_proj') or {}).get('gemv_us'))"
  done
done
