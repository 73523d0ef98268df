#!/bin/bash
# Same-box A/B of two source snapshots of csrc files: bash tools/ab_src.sh <dirA> <dirB> [rounds]
# (each dir holds the csrc/*.cu|*.h files that differ; they are copied over the tree before each build)
A=$1; B=$2; N=${3:-2}; C=paper_2511_10645_b200/csrc
for r in $(seq $N); do
  for v in $A $B; do
    cp $v/* $C/
    python -c "from importlib import util; import sys; sys.path.insert(0,'.'); spec=util.spec_from_file_location('b','paper_2511_10645_b200/_build.py'); m=util.module_from_spec(spec); spec.loader.exec_module(m); m.build(force=True)" > /dev/null 2>&1 || echo "BUILD FAIL $v"
    python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extra --no-prefill 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$v] step', d['us_per_step'], 'norot', d.get('us_per_step_norot'))"
  done
done
cp $B/* $C/
