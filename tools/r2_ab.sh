#!/bin/bash
mkdir -p gpurun_out/r2
for cfg in c2 c5 c4_8x; do
  for pf in 1 0; do
    echo "== $cfg prefetch $pf" >> gpurun_out/r2/ab_$1.txt
    KVP_PREFETCH_V=$pf timeout 120 python tools/kbench_fused.py --config $cfg --cluster 0 >> gpurun_out/r2/ab_$1.txt 2>&1
  done
done
KVP_PREFETCH_V=1 timeout 120 python tools/kbench_fused.py --config c2 --cluster 6 >> gpurun_out/r2/ab_$1.txt 2>&1
timeout 120 python tools/kbench_fused.py --config c2 --cluster 0 --trace >> gpurun_out/r2/ab_$1.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"qdots|core|vsum" -c 24 --csv --log-file gpurun_out/r2/launch_$1.csv python tools/kbench_fused.py --config c2 --cluster 0 --iters 1 --layers 4 > /dev/null 2>&1
