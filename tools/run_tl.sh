#!/bin/bash
for a in "4096 14336 rot 1" "14336 4096 rot 2" "4096 4096 rot 1"; do
  echo "== $a"; timeout 60 python tools/timeline.py $a 2>&1 | grep -v layer1
done
