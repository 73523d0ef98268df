#!/bin/bash
# Timeline (PARO_TIMELINE build) of one decode launch at B = 1, 4, 16 (Qwen3-4B MLP shapes).
export PARO_NVCC_EXTRA="-DPARO_TIMELINE=1 -DPARO_DEBUG_KNOBS=1"
python -c "import paper_2511_10645_b200._build as b; b.build(force=True)" > /dev/null 2>&1 || echo BUILD FAIL
for B in 1 4 16; do
  timeout 120 python tools/timeline_one.py 9728 2560 $B
  timeout 120 python tools/timeline_one.py 2560 9728 $B
done
