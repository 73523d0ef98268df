#!/bin/bash
timeout 300 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for env in "PARO_NW=8" ; do
  echo "== $env 4096"; env $env timeout 60 python tools/timeline.py 4096 4096 rot 1 2>&1 | grep -v layer1
  echo "== $env 14336x2 nomath"; env $env PARO_SKIP_MATH=1 timeout 60 python tools/timeline.py 14336 4096 rot 2 2>&1 | grep -v layer1
done
bash tools/run_combos.sh
