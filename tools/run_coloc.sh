#!/bin/bash
O=gpurun_out/coloc; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
run() { echo "== $*"; env "$@" PARO_PLAN_DEBUG=0 timeout 120 python tools/time_groups.py norot 1; env "$@" timeout 120 python tools/time_groups.py rot 1; }
{
run PARO_X=0
run PARO_NW=7 PARO_CTAS_PER_SM=3 PARO_CLUSTER=4
run PARO_NW=7 PARO_CTAS_PER_SM=3 PARO_CLUSTER=4 PARO_EARLY_STAGES=60
run PARO_NW=7 PARO_CTAS_PER_SM=3 PARO_CLUSTER=2 PARO_EARLY_STAGES=60
run PARO_NW=8 PARO_CTAS_PER_SM=3 PARO_CLUSTER=2 PARO_EARLY_STAGES=60
run PARO_NW=7 PARO_CTAS_PER_SM=3 PARO_CLUSTER=2 PARO_EARLY_STAGES=60 PARO_XFIRST=0
} > $O/sweep.txt 2>&1
PARO_PLAN_DEBUG=1 PARO_NW=7 PARO_CTAS_PER_SM=3 PARO_CLUSTER=2 timeout 120 python tools/time_groups.py norot 1 > $O/plan.txt 2>&1
echo done
