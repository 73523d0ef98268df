#!/bin/bash
O=gpurun_out/ab3; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
(cd _head && python -c "import __graft_entry__ as g; g.build()" > ../$O/build_head.txt 2>&1)
timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
for r in 1 2; do
  echo "== HEAD $r"; (cd _head && timeout 120 python tools/time_groups.py rot 1 && timeout 120 python tools/time_70b.py)
  echo "== WARM $r"; timeout 120 python tools/time_groups.py rot 1; timeout 120 python tools/time_70b.py
  echo "== NOWARM $r"; PARO_G1_WARM=0 timeout 120 python tools/time_groups.py rot 1 | tail -1
done > $O/ab.txt 2>&1
echo done
