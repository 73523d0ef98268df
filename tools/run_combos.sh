#!/bin/bash
for env in "PARO_CTAS_PER_SM=2" "PARO_CTAS_PER_SM=2 PARO_RG=2" "PARO_CTAS_PER_SM=1" "PARO_CTAS_PER_SM=1 PARO_CLUSTER=4" "PARO_CTAS_PER_SM=1 PARO_CLUSTER=2" "PARO_CTAS_PER_SM=2 PARO_CLUSTER=4"; do
  echo "== $env"; env $env timeout 120 python tools/time_groups.py rot 0
done
