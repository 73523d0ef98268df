#!/bin/bash
O=gpurun_out/ncu_g1; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:paro_gemv1 -s 2 -c 1 -f \
    -o $O/gateup python tools/prof_multi.py 14336,14336 4096 rot 4 > $O/ncu_gateup.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:paro_gemv1 -s 2 -c 1 -f \
    -o $O/oproj python tools/prof_multi.py 4096 4096 rot 4 > $O/ncu_oproj.log 2>&1
echo done
