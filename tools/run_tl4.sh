#!/bin/bash
O=gpurun_out/tl4; mkdir -p $O
PARO_NVCC_EXTRA=-DG1_TL=1 python -c "import sys; sys.path.insert(0,'paper_2511_10645_b200'); import _build; _build.build(force=True)" > $O/build_tl.txt 2>&1
for a in "4096 14336 rot" "4096 14336 norot" "4096,1024,1024 4096 rot"; do
  timeout 120 python tools/timeline1.py $a 2>&1 | tail -11
done > $O/tl.txt
PARO_G1_CL=4 timeout 120 python tools/timeline1.py 4096 14336 rot 2>&1 | tail -11 >> $O/tl.txt
echo done
