#!/bin/bash
for b in 1 8; do echo "== B=$b"; TL_B=$b timeout 60 python tools/timeline.py 4096 4096 rot 1 2>&1; done
timeout 120 python tools/time_groups.py rot 1
