#!/bin/bash
O=gpurun_out/g1l; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
{ timeout 120 python tools/time_groups.py rot 1; timeout 120 python tools/time_groups.py norot 1;
  for sh in "4096 4096" "14336 4096" "4096 14336" "9728 2560"; do timeout 120 python tools/time_batch.py $sh; done; } > $O/sweep.txt 2>&1
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
echo done
