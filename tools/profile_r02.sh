#!/bin/bash
# Round-2 profile: bench lines, ncu launch list of the bench, ncu --set full of each decode launch
# (B = 1), the B = 16 decode on both engines, the prefill GEMM and the FWHT.  -> gpurun_out/prof/
set -u
O=gpurun_out/prof; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --steps 200 --warmup 20 > $O/bench_long.json 2> $O/bench_long.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extra --no-prefill --load-s 0 > $O/bench_under_ncu.log 2>&1
i=0
for g in "4096,1024,1024 4096 1" "4096 4096 1" "14336,14336 4096 1" "4096 14336 1" "4096,1024,1024 2560 16" "4096,1024,1024 2560 16 tc" "8192 28672 1"; do
  set -- $g
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"paro_gemv1?(_b1)?_kernel" -s 2 -c 1 -f \
    -o $O/group$i python tools/prof_multi.py $1 $2 rot 4 $3 ${4:-} > $O/ncu_group$i.log 2>&1
  i=$((i+1))
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:prefill_gemm -s 1 -c 1 -f \
  -o $O/prefill_q python tools/ncu_prefill.py 4096 4096 2048 > $O/ncu_prefill.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:prefill_gemm -s 1 -c 1 -f \
  -o $O/prefill_gate python tools/ncu_prefill.py 14336 4096 2048 > $O/ncu_prefill_gate.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:transform_dense -s 1 -c 1 -f \
  -o $O/prefill_transform python tools/ncu_prefill.py 4096 4096 2048 > $O/ncu_prefill_transform.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/prefill_launches.csv \
  python tools/ncu_prefill.py 4096 4096 2048 3 > /dev/null 2>&1
echo done
