#!/bin/bash
# same-box A/B of prefill build variants: bash tools/ab_prefill.sh "<nvcc extra A>" "<nvcc extra B>" ...
for v in "$@"; do
  PARO_NVCC_EXTRA="$v" python -c "from importlib import util; import sys; sys.path.insert(0,'.'); spec=util.spec_from_file_location('b','paper_2511_10645_b200/_build.py'); m=util.module_from_spec(spec); spec.loader.exec_module(m); m.build(force=True)" > /dev/null 2>&1 || echo BUILD FAIL
  echo "== variant [$v]"; timeout 300 python tools/time_prefill.py 2048 | tail -${TAILN:-3}
done
