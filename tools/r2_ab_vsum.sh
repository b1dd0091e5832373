#!/bin/bash
mkdir -p gpurun_out/r2
T=$1
timeout 300 python tools/kbench_fused.py --config c2 > gpurun_out/r2/vsum_kb_$T.txt 2>&1
timeout 900 python bench.py > gpurun_out/r2/vsum_bench_$T.json 2> gpurun_out/r2/vsum_bench_$T.err
timeout 900 python bench.py --config c3 --steps 8 --no-cpu-baseline > gpurun_out/r2/c3_bench_$T.json 2> gpurun_out/r2/c3_bench_$T.err
