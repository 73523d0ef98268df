#!/bin/bash
# B = 2..4: cluster-shared-transform kernel (gemv.cu) vs the K-split kernel (PARO_G1_SMALLB=1).
export PARO_NVCC_EXTRA="-DPARO_DEBUG_KNOBS=1"
python -c "import paper_2511_10645_b200._build as b; b.build(force=True)" > /dev/null 2>&1 || { echo "BUILD FAIL"; exit 1; }
for sb in 0 1; do
  echo "=== PARO_G1_SMALLB=$sb"
  for s in "9728 2560" "2560 9728" "4096 4096" "28672 4096" "4096 14336" "1024 4096"; do
    TB_BATCHES=2,3,4 PARO_G1_SMALLB=$sb timeout 120 python tools/time_batch.py $s 2>&1 | grep -E "B=(2|3|4):"
  done
done
