#!/bin/bash
O=gpurun_out/tl2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 600 python -m pytest tests -x -q -m gpu > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
{
for pre in 2 0 1 4 99; do
  echo "== PRE=$pre"; PARO_G1_PRE=$pre PARO_G1_TPS=32 timeout 120 python tools/time_groups.py rot 1
done
echo "== PRE=2 TPS=16"; PARO_G1_PRE=2 PARO_G1_TPS=16 timeout 120 python tools/time_groups.py rot 1
echo "== PRE=2 TPS=32 norot"; PARO_G1_PRE=2 PARO_G1_TPS=32 timeout 120 python tools/time_groups.py norot 1
} > $O/sweep.txt 2>&1
PARO_NVCC_EXTRA=-DG1_TL=1 python -c "import sys; sys.path.insert(0,'paper_2511_10645_b200'); import _build; _build.build(force=True)" > $O/build_tl.txt 2>&1
for a in "4096 4096 rot" "14336,14336 4096 rot" "4096 14336 rot"; do
  PARO_G1_TPS=32 timeout 120 python tools/timeline1.py $a 2>&1 | tail -9
done > $O/tl.txt
echo done
