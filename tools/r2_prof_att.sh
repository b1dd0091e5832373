#!/bin/bash
# Decode-attention ncu at the bench's final tail (C2, 256 steps): per-kernel DRAM bytes + times for all
# layers, one full capture of the core kernel; plus the decode-step launch list of a short bench.
mkdir -p gpurun_out/r2
T=$1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/r2/att_tail_$T.csv python tools/ncu_tail.py c2 256 > gpurun_out/r2/att_tail_$T.log 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:'core_kernel|qdots|vsum' -c 3 \
  -o gpurun_out/r2/att_full_$T -f python tools/ncu_tail.py c2 256 > gpurun_out/r2/att_full_$T.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r2/launch_$T.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --factor-init placeholder > /dev/null 2>&1
