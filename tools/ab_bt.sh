#!/bin/bash
# B > 1 decode: parity tests, then launch times at the Qwen3-4B MLP and a 4096^2 shape.
timeout 300 python -m pytest -q -x tests/test_gpu_chain.py tests/test_gpu_parity.py -k "not llama" 2>&1 | tail -2
for s in "9728 2560" "2560 9728" "4096 4096"; do timeout 120 python tools/time_batch.py $s 2>&1 | grep -v "^\[paro"; done
