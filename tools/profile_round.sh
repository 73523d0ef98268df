#!/bin/bash
# Round profile: bench line, ncu launch list of the bench, ncu --set full of each decode group.
# Output under gpurun_out/prof/ (copy the summaries into profiles/rNN/).
set -u
O=gpurun_out/prof; mkdir -p $O
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --load-s 0 > $O/bench_under_ncu.log 2>&1
i=0
for g in "4096,1024,1024 4096" "4096 4096" "14336,14336 4096" "4096 14336"; do
  set -- $g
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:paro_gemv -s 2 -c 1 -f \
    -o $O/group$i python tools/prof_multi.py $1 $2 rot 4 > $O/ncu_group$i.log 2>&1
  i=$((i+1))
done
echo done
