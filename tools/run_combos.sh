#!/bin/bash
# decode-kernel config sweep (graph timing of the bench's launch groups)
for env in "PARO_NW=8 PARO_CLUSTER=8" "PARO_NW=8 PARO_CLUSTER=4" "PARO_NW=16 PARO_CLUSTER=4 PARO_TPS=32" "PARO_NW=16 PARO_CLUSTER=2 PARO_TPS=32"; do
  echo "== $env"; env $env timeout 120 python tools/time_groups.py rot 0 2>&1
done
