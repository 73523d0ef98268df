#!/bin/bash
O=gpurun_out/g1g; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
{ timeout 120 python tools/time_groups.py rot 1; timeout 120 python tools/time_groups.py norot 1; } > $O/sweep.txt 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
echo done
