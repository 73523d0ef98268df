#!/bin/bash
# decode-linear graph timings for the LLaMA-3-8B shapes
python tools/empty_graph.py
for nk in "4096 4096" "1024 4096" "14336 4096" "4096 14336"; do for m in norot rot; do timeout 60 python tools/time_graph.py $nk $m 1 100; done; done
