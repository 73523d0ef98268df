#!/bin/bash
O=gpurun_out/g1n; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
{ timeout 120 python tools/time_groups.py rot 1; timeout 120 python tools/time_groups.py norot 1;
  echo "== TPS32"; PARO_G1_TPS=32 timeout 120 python tools/time_groups.py rot 1;
  echo "== TPS24"; PARO_G1_TPS=24 timeout 120 python tools/time_groups.py rot 1;
  for sh in "4096 4096" "14336 4096"; do timeout 120 python tools/time_batch.py $sh; done; } > $O/sweep.txt 2>&1
PARO_PLAN_DEBUG=1 timeout 120 python tools/time_groups.py rot 1 2>&1 | grep plan | sort -u > $O/plan.txt
echo done
