#!/bin/bash
O=gpurun_out/g1f; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 600 python -m pytest tests -x -q -m gpu > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
{
for sh in "4096 4096" "14336 4096" "4096 14336" "9728 2560"; do
  echo "== $sh gemv1"; timeout 120 python tools/time_batch.py $sh
  echo "== $sh old"; PARO_GEMV1=0 timeout 120 python tools/time_batch.py $sh
done
echo "== layer"; timeout 120 python tools/time_groups.py rot 1
} > $O/sweep.txt 2>&1
echo done
