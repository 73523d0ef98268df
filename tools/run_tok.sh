#!/bin/bash
O=gpurun_out/tok; mkdir -p $O
for cfg in "8 4" "8 8" "16 8" "16 4" "4 4"; do set -- $cfg
  PARO_NVCC_EXTRA="-DPARO_TOK_PER_WARP=$1 -DPARO_TOK_LOCK=$2" python -c "import sys; sys.path.insert(0,'paper_2511_10645_b200'); import _build; _build.build(force=True)" > $O/build.txt 2>&1
  echo "== per_warp=$1 lock=$2"; for k in 4096 14336; do timeout 60 python tools/time_transform.py $k 2048; done
done > $O/a.txt 2>&1
echo done
