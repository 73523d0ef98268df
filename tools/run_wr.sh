#!/bin/bash
O=gpurun_out/wr; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
for r in 1 2; do
{ echo "== wring"; PARO_PLAN_DEBUG=1 timeout 120 python tools/time_groups.py rot 1 2>&1 | sort -u; timeout 120 python tools/time_70b.py;
  echo "== stage ring"; PARO_G1_WRING=0 timeout 120 python tools/time_groups.py rot 1; PARO_G1_WRING=0 timeout 120 python tools/time_70b.py; } >> $O/a.txt 2>&1
done
echo done
