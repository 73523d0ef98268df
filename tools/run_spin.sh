#!/bin/bash
O=gpurun_out/spin; mkdir -p $O
PARO_NVCC_EXTRA="-DPARO_MBAR_SPIN=1" python -c "import sys; sys.path.insert(0,'paper_2511_10645_b200'); import _build; _build.build(force=True)" > $O/build.txt 2>&1
for t in 32 16; do echo "== SPIN TPS=$t"; PARO_G1_TPS=$t timeout 120 python tools/time_70b.py 2>&1; PARO_G1_TPS=$t timeout 120 python tools/time_groups.py rot 1; done > $O/a.txt 2>&1
echo done
