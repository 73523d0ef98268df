#!/bin/bash
O=gpurun_out/ldg; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
PARO_G1_LDG=1 timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
{ echo "== ring"; timeout 120 python tools/time_groups.py rot 1; timeout 120 python tools/time_70b.py;
  for ah in 6 16 2; do echo "== LDG ahead=$ah"; PARO_G1_LDG=1 PARO_G1_LDG_AHEAD=$ah timeout 120 python tools/time_groups.py rot 1; PARO_G1_LDG=1 PARO_G1_LDG_AHEAD=$ah timeout 120 python tools/time_70b.py; done; } > $O/a.txt 2>&1
echo done
