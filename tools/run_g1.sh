#!/bin/bash
O=gpurun_out/g1; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 600 python -m pytest tests -x -q -m gpu > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
run() { echo "== $*"; env "$@" timeout 120 python tools/time_groups.py norot 1; env "$@" timeout 120 python tools/time_groups.py rot 1; }
{
run PARO_GEMV1=0
run PARO_GEMV1=1
run PARO_G1_CL=4
run PARO_G1_CL=8
run PARO_G1_TPS=32
run PARO_G1_TPS=8
} > $O/sweep.txt 2>&1
PARO_PLAN_DEBUG=1 timeout 120 python tools/time_groups.py rot 1 2>&1 | sort -u | grep plan > $O/plan.txt
echo done
