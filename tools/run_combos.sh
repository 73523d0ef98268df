#!/bin/bash
for env in "PARO_NW=15" "PARO_NW=15 PARO_TPS=45"; do
  echo "== $env"; env $env timeout 120 python tools/time_groups.py rot 1 2>&1
done
timeout 120 python tools/time_groups.py norot 1 2>&1
timeout 60 python tools/timeline.py 4096 14336 rot 1 2>&1 | grep -v layer1
timeout 60 python tools/timeline.py 4096 4096 rot 1 2>&1 | grep -v layer1
