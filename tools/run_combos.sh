#!/bin/bash
PARO_NVCC_EXTRA="-DPARO_ENABLE_DEBUG=1" python -c "from paper_2511_10645_b200 import _build; _build.build(force=True)"
timeout 60 python tools/timeline.py 4096 4096 rot 1 2>&1
