#!/bin/bash
# env-knob sweep of the decode launch groups (release build)
O=gpurun_out/sweep; mkdir -p $O; : > $O/sweep.txt
run() { echo "== $*" >> $O/sweep.txt; env "$@" timeout 120 python tools/time_groups.py rot 1 >> $O/sweep.txt 2>&1; }
run PARO_IMMA=1
run PARO_SKIP_MATH=1
run PARO_STAGGER=0
run PARO_XFIRST=0
run PARO_EARLY_STAGES=0
run PARO_EARLY_STAGES=4
run PARO_TPS=8
run PARO_TPS=16
run PARO_TPS=48
run PARO_CLUSTER=2
run PARO_CLUSTER=1
run PARO_NW=8
run PARO_NW=12
run PARO_NW=19
