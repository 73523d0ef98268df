#!/bin/bash
# same-box A/B of decode build variants at B > 1 (tools/ncu_batch.py timings, Qwen3-4B shapes):
# bash tools/ab_batch.sh "<nvcc extra A>" "<nvcc extra B>" ...
for v in "$@"; do
  PARO_NVCC_EXTRA="$v" python -c "from importlib import util; import sys; sys.path.insert(0,'.'); spec=util.spec_from_file_location('b','paper_2511_10645_b200/_build.py'); m=util.module_from_spec(spec); spec.loader.exec_module(m); m.build(force=True)" > /dev/null 2>&1 || echo BUILD FAIL
  echo "== variant [$v]"
  for B in ${BS:-2 4 8 16}; do for w in qkv gateup down; do timeout 120 python tools/ncu_batch.py $B $w; done; done
done
