#!/bin/bash
echo "== debug compiled in"; timeout 120 python tools/time_groups.py rot 1
PARO_NVCC_EXTRA="-DPARO_ENABLE_DEBUG=0" python -c "from paper_2511_10645_b200 import _build; _build.build(force=True)"
echo "== debug compiled out"; timeout 120 python tools/time_groups.py rot 1
cuobjdump -sass -fun '_ZN4paro16paro_gemv_kernelILi1ELi512EEEvNS_8GemvArgsE' paper_2511_10645_b200/libparo.so | grep -c "^        /\*[0-9a-f]*\*/"
