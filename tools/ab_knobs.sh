#!/bin/bash
# One debug-knob build, then the 4-launch step (tools/ab_step.py) under each knob setting.
# Usage: KNOBS="PARO_G1_TPS=28|PARO_G1_TPS=24,PARO_G1_PRE=3" bash tools/ab_knobs.sh
export PARO_NVCC_EXTRA="-DPARO_DEBUG_KNOBS=1 $EXTRA"
python -c "from importlib import util; import sys; sys.path.insert(0,'.'); spec=util.spec_from_file_location('b','paper_2511_10645_b200/_build.py'); m=util.module_from_spec(spec); spec.loader.exec_module(m); m.build(force=True)" > /dev/null 2>&1 || { echo "BUILD FAIL"; exit 1; }
IFS='|' read -ra KS <<< "${KNOBS}"
for k in "" "${KS[@]}"; do
  echo "=== knobs: '$k'"
  env $(echo $k | tr ',' ' ') python tools/ab_step.py . 2>&1 | grep -v package
done
