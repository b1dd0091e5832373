#!/bin/bash
mkdir -p gpurun_out/r2
T=$1
KVP_TRACE_COMPACT=1 timeout 600 python tools/tcompact.py c2 8 2 > gpurun_out/r2/ctime_$T.txt 2>&1
KVP_TRACE_COMPACT=1 timeout 600 python tools/tcompact.py c3 3 2 >> gpurun_out/r2/ctime_$T.txt 2>&1
timeout 600 python tools/check_compaction.py 4096 5120 284 1 >> gpurun_out/r2/ctime_$T.txt 2>&1
