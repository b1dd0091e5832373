#!/bin/bash
mkdir -p gpurun_out/r2
T=$1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r2/ctime_$T.txt 2>&1
lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/r2/ctime_$T.txt 2>&1
KVP_TRACE_COMPACT=1 timeout 600 python tools/tcompact.py c2 32 3 >> gpurun_out/r2/ctime_$T.txt 2>&1
timeout 600 python tools/check_compaction.py 2304 4096 368 1 >> gpurun_out/r2/ctime_$T.txt 2>&1
timeout 600 python tools/check_compaction.py 4096 4096 1024 1 >> gpurun_out/r2/ctime_$T.txt 2>&1
KVP_TRACE_COMPACT=1 timeout 600 python tools/tcompact.py c3 3 2 >> gpurun_out/r2/ctime_$T.txt 2>&1
