#!/bin/bash
mkdir -p gpurun_out/r2
T=$1
timeout 600 python tools/tcompact.py c2 32 4 > gpurun_out/r2/lanes_$T.txt 2>&1
timeout 300 python tools/check_compaction.py 2304 4096 368 1 >> gpurun_out/r2/lanes_$T.txt 2>&1
