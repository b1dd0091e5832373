#!/bin/bash
mkdir -p gpurun_out/r2
timeout 120 python tools/kbench_fused.py --config c2 --cluster 0 --trace > gpurun_out/r2/trace_$1.txt 2>&1
timeout 120 python tools/kbench_fused.py --config c2 --cluster 6 --trace >> gpurun_out/r2/trace_$1.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"qdots|core|vsum" -c 24 --csv --log-file gpurun_out/r2/launch_$1.csv python tools/kbench_fused.py --config c2 --cluster 0 --iters 1 --layers 4 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"qdots|core|vsum" -c 24 --csv --log-file gpurun_out/r2/launch6_$1.csv python tools/kbench_fused.py --config c2 --cluster 6 --iters 1 --layers 4 > /dev/null 2>&1
