#!/bin/bash
O=gpurun_out/tl1; mkdir -p $O
PARO_NVCC_EXTRA=-DG1_TL=1 python -c "import sys; sys.path.insert(0,'paper_2511_10645_b200'); import _build; _build.build(force=True)" > $O/build.txt 2>&1
for tps in 16 32; do
for a in "4096 4096 norot" "4096 4096 rot" "14336,14336 4096 rot" "4096 14336 rot" "4096,1024,1024 4096 rot"; do
  PARO_G1_TPS=$tps timeout 120 python tools/timeline1.py $a 2>&1 | tail -9
done; done > $O/tl.txt
echo done
