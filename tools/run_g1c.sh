#!/bin/bash
O=gpurun_out/g1c; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
{
echo "== NW16 TPS32"; timeout 120 python tools/time_groups.py rot 1
echo "== NW8 CL2"; PARO_G1_NW=8 timeout 120 python tools/time_groups.py rot 1
echo "== NW8 CL2 norot"; PARO_G1_NW=8 timeout 120 python tools/time_groups.py norot 1
echo "== NW8 CL4"; PARO_G1_NW=8 PARO_G1_CL=4 timeout 120 python tools/time_groups.py rot 1
echo "== NW8 CL2 PRE8"; PARO_G1_NW=8 PARO_G1_PRE=8 timeout 120 python tools/time_groups.py rot 1
echo "== NW8 CL2 TPS8"; PARO_G1_NW=8 PARO_G1_TPS=8 timeout 120 python tools/time_groups.py rot 1
} > $O/sweep.txt 2>&1
PARO_PLAN_DEBUG=1 PARO_G1_NW=8 timeout 120 python tools/time_groups.py rot 1 2>&1 | grep plan | sort -u > $O/plan.txt
PARO_G1_NW=8 timeout 600 python -m pytest tests -x -q -m gpu > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
echo done
