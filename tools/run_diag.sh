#!/bin/bash
# Diagnostics: group timings (release build), then per-CTA timelines (debug build).
O=gpurun_out/diag; mkdir -p $O
timeout 300 python tools/time_groups.py rot 1 > $O/groups_rot_pdl.txt 2>&1
timeout 300 python tools/time_groups.py norot 1 > $O/groups_norot_pdl.txt 2>&1
timeout 300 python tools/time_groups.py rot 0 > $O/groups_rot_nopdl.txt 2>&1
PARO_NVCC_EXTRA=-DPARO_ENABLE_DEBUG=1 python -c "import __graft_entry__ as g; g.build()" > $O/build_dbg.txt 2>&1
touch paper_2511_10645_b200/csrc/gemv.cu
PARO_NVCC_EXTRA=-DPARO_ENABLE_DEBUG=1 python paper_2511_10645_b200/_build.py -f >> $O/build_dbg.txt 2>&1
for a in "14336 4096 rot 1" "14336 4096 rot 2" "14336 4096 norot 1" "4096 4096 rot 1" "1024 4096 rot 1" "4096 14336 rot 1"; do
  echo "== $a" >> $O/timeline.txt
  timeout 120 python tools/timeline.py $a >> $O/timeline.txt 2>&1
done
