#!/bin/bash
O=gpurun_out/nw; mkdir -p $O
for nw in 16 24 20; do
  PARO_NVCC_EXTRA="-DG1_NWARPS=$nw" python -c "import sys; sys.path.insert(0,'paper_2511_10645_b200'); import _build; _build.build(force=True)" > $O/build_$nw.txt 2>&1
  { echo "== NW=$nw"; timeout 120 python tools/time_groups.py rot 1; timeout 120 python tools/time_70b.py; timeout 120 python tools/time_batch.py 4096 4096; } >> $O/a.txt 2>&1
done
timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest20.txt 2>&1; echo "rc=$?" >> $O/pytest20.txt
echo done
