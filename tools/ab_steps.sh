#!/bin/bash
# Same-box A/B of several compile-time variants on the decode step only:
#   bash tools/ab_steps.sh "<flags A>" "<flags B>" ...   (ROUNDS env, default 2)
for r in $(seq ${ROUNDS:-2}); do
  for v in "$@"; do
    PARO_NVCC_EXTRA="$v" python -c "from importlib import util; import sys; sys.path.insert(0,'.'); spec=util.spec_from_file_location('b','paper_2511_10645_b200/_build.py'); m=util.module_from_spec(spec); spec.loader.exec_module(m); m.build(force=True)" > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
    python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extra --no-prefill 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$v] step', d['us_per_step'], 'norot', d.get('us_per_step_norot'))"
  done
done
