#!/bin/bash
O=gpurun_out/imma; mkdir -p $O
timeout 600 python -m pytest tests -x -q -m gpu > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
for m in 1 0; do
  PARO_IMMA=$m timeout 300 python tools/time_groups.py rot 1 > $O/groups_rot_imma$m.txt 2>&1
  PARO_IMMA=$m timeout 300 python tools/time_groups.py norot 1 > $O/groups_norot_imma$m.txt 2>&1
done
