#!/bin/bash
# One GPU-box pass: build, pytest -m gpu, compute-sanitizer over tools/sanitize_cases.py, short bench.
# Usage (from gpurun): bash tools/gpu_check.sh [tag]   -> gpurun_out/<tag>/...
TAG=${1:-check}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
if [ -z "$NO_SAN" ]; then
for tool in memcheck racecheck synccheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py --quick > $OUT/sanitize_$tool.log 2>&1
  echo "rc=$?" >> $OUT/sanitize_$tool.log
done
fi
timeout 900 python bench.py --steps 200 --warmup 20 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
tail -3 $OUT/pytest_gpu.log
