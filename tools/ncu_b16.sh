mkdir -p gpurun_out/b16
for B in 1 4 8 16; do for w in qkv gateup down; do python tools/ncu_batch.py $B $w; done; done > gpurun_out/b16/times.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:paro_gemv1_kernel -s 10 -c 1 -o gpurun_out/b16/qkv16 -f python tools/ncu_batch.py 16 qkv > gpurun_out/b16/ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/b16/qkv16.ncu-rep > gpurun_out/b16/qkv16_summary.txt 2>&1
cat gpurun_out/b16/times.txt; head -40 gpurun_out/b16/qkv16_summary.txt
