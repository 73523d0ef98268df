#!/bin/bash
O=gpurun_out/g1h; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
{
echo "== PF1"; timeout 120 python tools/time_groups.py rot 1
echo "== PF0"; PARO_G1_PF=0 timeout 120 python tools/time_groups.py rot 1
echo "== PF1 PRE4"; PARO_G1_PRE=4 timeout 120 python tools/time_groups.py rot 1
echo "== PF1 PRE1"; PARO_G1_PRE=1 timeout 120 python tools/time_groups.py rot 1
} > $O/sweep.txt 2>&1
PARO_NVCC_EXTRA=-DG1_TL=1 python -c "import sys; sys.path.insert(0,'paper_2511_10645_b200'); import _build; _build.build(force=True)" > $O/build_tl.txt 2>&1
for a in "4096 4096 rot" "4096 4096 norot"; do
  timeout 120 python tools/timeline1.py $a 2>&1 | tail -9
done > $O/tl.txt
echo done
