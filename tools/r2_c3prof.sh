#!/bin/bash
mkdir -p gpurun_out/r2
T=$1
timeout 600 python tools/tcompact.py c2 32 3 > gpurun_out/r2/c2t_$T.txt 2>&1
timeout 600 python tools/tcompact.py c3 3 > gpurun_out/r2/c3t_$T.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2/c3_launch_$T.csv python tools/tcompact.py c3 1 > /dev/null 2>&1
timeout 600 python tools/tcompact.py c4_2x 2 >> gpurun_out/r2/c3t_$T.txt 2>&1
