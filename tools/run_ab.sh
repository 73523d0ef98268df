#!/bin/bash
# A/B: committed HEAD (in _head/) vs working tree, same box, interleaved
O=gpurun_out/ab; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
(cd _head && python -c "import __graft_entry__ as g; g.build()" > ../$O/build_head.txt 2>&1)
for r in 1 2; do
  echo "== HEAD run $r"; (cd _head && timeout 120 python tools/time_groups.py rot 1)
  echo "== WORK run $r"; timeout 120 python tools/time_groups.py rot 1
done > $O/ab.txt 2>&1
echo done
