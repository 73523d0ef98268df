#!/bin/bash
# per-CTA timeline of the bench step (tools/timeline_b1.py) with a PARO_TIMELINE build
export PARO_NVCC_EXTRA="-DPARO_TIMELINE=1"
python -c "from importlib import util; import sys; sys.path.insert(0,'.'); spec=util.spec_from_file_location('b','paper_2511_10645_b200/_build.py'); m=util.module_from_spec(spec); spec.loader.exec_module(m); m.build(force=True)" > /dev/null 2>&1 || echo BUILD FAIL
timeout 300 python tools/timeline_b1.py
