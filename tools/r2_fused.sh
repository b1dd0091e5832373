#!/bin/bash
# Fused-kernel parity + split vs cluster timing on one box.
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_parity_configs.py -q -rA -s -k "fused" > gpurun_out/r2/fused_$1.txt 2>&1
for cfg in c2 c4_8x c5 c4_2x c3; do
  for cl in 0 6 8; do
    echo "== $cfg cluster $cl" >> gpurun_out/r2/kb_$1.txt
    timeout 120 python tools/kbench_fused.py --config $cfg --cluster $cl >> gpurun_out/r2/kb_$1.txt 2>&1
  done
done
timeout 120 python tools/kbench_fused.py --config c2 --cluster 0 --trace >> gpurun_out/r2/kb_$1.txt 2>&1
timeout 300 python bench.py --steps 30 > gpurun_out/r2/bench_$1.json 2> gpurun_out/r2/bench_$1.err
