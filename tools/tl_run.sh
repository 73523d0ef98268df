#!/bin/bash
# Timeline experiments (debug-knob + timeline build): chain at several plans, and the 4-launch form.
export PARO_NVCC_EXTRA="-DPARO_TIMELINE=1 -DPARO_DEBUG_KNOBS=1"
python -c "from importlib import util; import sys; sys.path.insert(0,'.'); spec=util.spec_from_file_location('b','paper_2511_10645_b200/_build.py'); m=util.module_from_spec(spec); spec.loader.exec_module(m); m.build(force=True)" > /dev/null 2>&1 || echo BUILD FAIL
for cfg in ${CFGS:-"PARO_G1_CHAIN_CL=4"}; do echo "== $cfg"; env $(echo $cfg | tr ',' ' ') timeout 120 python tools/timeline_chain.py chain; done
echo "== multi"; timeout 120 python tools/timeline_chain.py multi
