#!/bin/bash
O=gpurun_out/g1b; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 600 python -m pytest tests -x -q -m gpu > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
run() { echo "== $*"; env "$@" timeout 120 python tools/time_groups.py norot 1; env "$@" timeout 120 python tools/time_groups.py rot 1; }
{
run PARO_GEMV1=1
run PARO_G1_TPS=32
run PARO_G1_CL=4
run PARO_G1_CL=4 PARO_G1_TPS=32
} > $O/sweep.txt 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:paro_gemv1 -s 2 -c 1 -f \
    -o $O/gateup python tools/prof_multi.py 14336,14336 4096 rot 4 > $O/ncu_gateup.log 2>&1
echo done
