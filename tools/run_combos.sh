#!/bin/bash
for t in 30 24 20 18 15; do echo "== TPS=$t"; PARO_TPS=$t PARO_PLAN_DEBUG=1 timeout 120 python tools/time_groups.py rot 1 2>&1 | sort -u | grep -v "^$" | grep "layer\|gate\|down\|o_proj\|q_proj\|K=4096 grid=148\|K=14336"; done
