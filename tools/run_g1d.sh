#!/bin/bash
O=gpurun_out/g1d; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 600 python -m pytest tests -x -q -m gpu > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
{
echo "== default"; timeout 120 python tools/time_groups.py rot 1; timeout 120 python tools/time_groups.py norot 1
echo "== PRE1"; PARO_G1_PRE=1 timeout 120 python tools/time_groups.py rot 1
echo "== TPS15"; PARO_G1_TPS=15 timeout 120 python tools/time_groups.py rot 1
echo "== CL2 all"; PARO_G1_CL=2 timeout 120 python tools/time_groups.py rot 1
} > $O/sweep.txt 2>&1
PARO_NVCC_EXTRA=-DG1_TL=1 python -c "import sys; sys.path.insert(0,'paper_2511_10645_b200'); import _build; _build.build(force=True)" > $O/build_tl.txt 2>&1
for a in "4096 4096 rot" "14336,14336 4096 rot" "4096 14336 rot"; do
  timeout 120 python tools/timeline1.py $a 2>&1 | tail -9
done > $O/tl.txt
echo done
