#!/bin/bash
# Follow-up GPU pass: synccheck of the chain cases, torchrun N-shard parity at world = 1, the B = 16
# GEMV captures (both engines), the chain timeline, and a bench line.  -> gpurun_out/r02b/
O=gpurun_out/r02b; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for c in chain_b1 chain_b4; do
  echo "=== synccheck $c" >> $O/sanitize_synccheck_chain.log
  timeout 300 /usr/local/cuda/bin/compute-sanitizer --tool synccheck --print-limit 10 python tools/sanitize_cases.py $c >> $O/sanitize_synccheck_chain.log 2>&1
  echo "rc=$?" >> $O/sanitize_synccheck_chain.log
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 tools/torchrun_parity.py > $O/torchrun_parity_w1.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 tools/torchrun_parity.py 8192 28672 3 >> $O/torchrun_parity_w1.log 2>&1
i=4
for g in "4096,1024,1024 2560 16" "4096,1024,1024 2560 16 tc"; do
  set -- $g
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:paro_gemv1_kernel -s 2 -c 1 -f \
    -o $O/group$i python tools/prof_multi.py $1 $2 rot 4 $3 ${4:-} > $O/ncu_group$i.log 2>&1
  i=$((i+1))
done
PARO_NVCC_EXTRA="-DPARO_TIMELINE=1" python -c "from importlib import util; spec=util.spec_from_file_location('b','paper_2511_10645_b200/_build.py'); m=util.module_from_spec(spec); spec.loader.exec_module(m); m.build(force=True)" > /dev/null 2>&1
timeout 120 python tools/timeline_chain.py chain > $O/chain_timeline.txt 2>&1
timeout 120 python tools/timeline_chain.py multi >> $O/chain_timeline.txt 2>&1
python -c "from importlib import util; spec=util.spec_from_file_location('b','paper_2511_10645_b200/_build.py'); m=util.module_from_spec(spec); spec.loader.exec_module(m); m.build(force=True)" > /dev/null 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err
tail -3 $O/torchrun_parity_w1.log; grep -E "ERROR SUMMARY|rc=" $O/sanitize_synccheck_chain.log
