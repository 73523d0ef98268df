#!/bin/bash
for env in "" "PARO_CTAS_PER_SM=1" "PARO_CLUSTER=2" "PARO_CLUSTER=4"; do
echo "== $env"
for nk in "4096 4096" "14336 4096" "4096 14336"; do for m in norot rot; do env $env timeout 60 python tools/time_graph.py $nk $m 1 100; done; done
done
