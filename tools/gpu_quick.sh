#!/bin/bash
# Quick GPU pass: build, the named test files (default: all -m gpu), a driver-style bench.
# Usage (from gpurun): bash tools/gpu_quick.sh <tag> [pytest targets...]   -> gpurun_out/<tag>/...
TAG=${1:-quick}; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
TARGETS=${@:-tests}
timeout 1500 python -m pytest $TARGETS -m gpu -q -p no:cacheprovider --timeout=300 -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -5 $OUT/pytest_gpu.log
if [ -z "$NO_BENCH" ]; then
  timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
  tail -3 $OUT/bench.err
  python -c "
import json,sys
d=json.loads(open('$OUT/bench.json').read().strip().splitlines()[-1])
for k in ('value','us_per_step','us_per_step_norot','rotation_overhead','us_per_step_4_launches','cold_step_us','frac_of_8TBps'): print(k, d.get(k))
print('e2e', d['e2e']['value'], d['e2e']['ms_per_step'])
print('c1', d.get('c1')); print('c3', d.get('c3_qwen3_4b_stack')); print('c5', json.dumps(d.get('c5_llama3_70b_mlp')))
print('prefill', d['prefill']['TFLOPs'] if d.get('prefill') else None)
print('per_linear', json.dumps(d.get('per_linear')))
print('fwht', json.dumps(d.get('transform_vs_fwht')))
" 2>&1 | tee $OUT/bench_summary.txt
fi
