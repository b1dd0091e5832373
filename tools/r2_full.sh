#!/bin/bash
# GPU-box round check: -m gpu suite, smoke, default bench line, launch list of a short bench.
# usage: tools/r2_full.sh TAG
mkdir -p gpurun_out/r2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2/gpu_$1.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rA -x > gpurun_out/r2/tests_$1.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2/smoke_$1.txt 2>&1
timeout 900 python bench.py > gpurun_out/r2/bench_$1.json 2> gpurun_out/r2/bench_$1.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 600 --csv --log-file gpurun_out/r2/launch_$1.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
  --factor-init placeholder > /dev/null 2>&1
