#!/bin/bash
# Per-CTA timelines of a q_proj-shaped B = 1 launch: the round-1 kernel (tmp_r1, -DG1_TL=1) vs now
# (-DPARO_TIMELINE=1).  Both libraries are rebuilt here with their timeline flags.
cd tmp_r1 && PARO_NVCC_EXTRA="-DG1_TL=1" python -c "from importlib import util; spec=util.spec_from_file_location('b','paper_2511_10645_b200/_build.py'); m=util.module_from_spec(spec); spec.loader.exec_module(m); m.build(force=True)" > /dev/null 2>&1 || echo R1 BUILD FAIL
cd ..
echo "== round 1"; PARO_PKG_DIR=tmp_r1 python tools/timeline1.py ${NS:-4096} 4096 rot
PARO_NVCC_EXTRA="-DPARO_TIMELINE=1" python -c "from importlib import util; import sys; spec=util.spec_from_file_location('b','paper_2511_10645_b200/_build.py'); m=util.module_from_spec(spec); spec.loader.exec_module(m); m.build(force=True)" > /dev/null 2>&1 || echo BUILD FAIL
echo "== now"; python tools/timeline_one.py ${NS:-4096} 4096 1
