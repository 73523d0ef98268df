#!/bin/bash
# Round check: GPU parity suite, bench line, per-group timings.
O=gpurun_out/check; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 300 python tools/time_groups.py rot 1 > $O/groups_rot.txt 2>&1
timeout 300 python tools/time_groups.py norot 1 > $O/groups_norot.txt 2>&1
echo done
