#!/bin/bash
# compute-sanitizer over tools/sanitize_cases.py, one process per (tool, case) with its own timeout.
# Usage (from gpurun): bash tools/gpu_sanitize.sh <tag> [tools...]  -> gpurun_out/<tag>/sanitize_<tool>.log
TAG=${1:-san}; shift
TOOLS=${@:-memcheck racecheck synccheck}
OUT=gpurun_out/$TAG; mkdir -p $OUT
CASES=${CASES:-"c1 q_b1_pdl q_b3 q_b2 q_b16 otf_b5 otf_b1 prefill_b300 dense copy multi chain_b1 chain_b4 q_b8_tcgen05"}
for tool in $TOOLS; do
  for c in $CASES; do
    echo "=== $tool $c" >> $OUT/sanitize_$tool.log
    timeout 240 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py $c >> $OUT/sanitize_$tool.log 2>&1
    echo "rc=$?" >> $OUT/sanitize_$tool.log
  done
  grep -E "^===|ERROR SUMMARY|rc=" $OUT/sanitize_$tool.log | paste - - - | tail -20
done
