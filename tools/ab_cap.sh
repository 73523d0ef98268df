for v in 0 1 0 1; do
  PARO_NVCC_EXTRA="-DPARO_B1_SHORT_MULTI_CAP=$v" python -c "from importlib import util; import sys; sys.path.insert(0,'.'); spec=util.spec_from_file_location('b','paper_2511_10645_b200/_build.py'); m=util.module_from_spec(spec); spec.loader.exec_module(m); m.build(force=True)" > /dev/null 2>&1
  echo "== cap=$v"; python tools/ab_step.py . 2>&1 | grep -E "step \(4"
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', d['us_per_step'], 'qwen bs1', d['c3_qwen3_4b_stack']['bs1']['us_per_step'])"
done
