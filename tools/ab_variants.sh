#!/bin/bash
# Build the library with each compile-time variant in turn and time the 4-launch step (tools/ab_step.py).
# Usage: VARIANTS="-DX=1|-DY=2" bash tools/ab_variants.sh
IFS='|' read -ra VS <<< "${VARIANTS}"
for v in "" "${VS[@]}"; do
  export PARO_NVCC_EXTRA="$v"
  python -c "from importlib import util; import sys; sys.path.insert(0,'.'); spec=util.spec_from_file_location('b','paper_2511_10645_b200/_build.py'); m=util.module_from_spec(spec); spec.loader.exec_module(m); m.build(force=True)" > /dev/null 2>&1 || { echo "BUILD FAIL $v"; continue; }
  echo "=== variant: '$v'"
  python tools/ab_step.py . 2>&1 | grep -v package
done
