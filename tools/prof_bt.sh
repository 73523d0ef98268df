#!/bin/bash
# Launch list + one full ncu capture of the B > 1 decode kernel (Qwen3-4B down-proj shape).
mkdir -p gpurun_out
B=${B:-16}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bt${B}_launches.csv python tools/prof_multi.py 9728 2560 rot 6 $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:paro_gemv1 -s 3 -c 1 -o gpurun_out/bt${B}_full -f python tools/prof_multi.py 9728 2560 rot 6 $B > /dev/null 2>&1
ls -la gpurun_out
