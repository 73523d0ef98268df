#!/bin/bash
O=gpurun_out/diag2; mkdir -p $O
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/probe_dot tools/probe_dot.cu && /tmp/probe_dot > $O/probe_dot.txt 2>&1
PARO_NVCC_EXTRA=-DPARO_ENABLE_DEBUG=1 python -c "import sys; sys.path.insert(0,'paper_2511_10645_b200'); import _build; _build.build(force=True)" > $O/build.txt 2>&1
for a in "4096 4096 norot 1" "4096 4096 rot 1" "14336 4096 norot 2" "4096 14336 rot 1"; do
  echo "== $a"; timeout 60 python tools/timeline.py $a 2>&1 | grep -v layer1
done > $O/timeline.txt
echo done
