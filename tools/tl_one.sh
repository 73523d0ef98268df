#!/bin/bash
export PARO_NVCC_EXTRA="-DPARO_TIMELINE=1 -DPARO_DEBUG_KNOBS=1"
python -c "from importlib import util; import sys; sys.path.insert(0,'.'); spec=util.spec_from_file_location('b','paper_2511_10645_b200/_build.py'); m=util.module_from_spec(spec); spec.loader.exec_module(m); m.build(force=True)" > /dev/null 2>&1 || echo BUILD FAIL
for c in ${CASES:-"4096 14336 4"}; do timeout 120 python tools/timeline_one.py $(echo $c | tr ',' ' ' | awk '{print $1" "$2" "$3}'); done
