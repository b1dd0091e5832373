#!/bin/bash
mkdir -p gpurun_out/r2
T=$1
{
timeout 600 python -m pytest tests/test_kvpack_api.py tests/test_gpu_parity_configs.py tests/test_gpu_engine.py -k "svd or singular or variance or compaction" -m gpu -q 2>&1 | tail -5
timeout 300 python tools/check_compaction.py 2304 4096 368 1
timeout 300 python tools/check_compaction.py 4096 4096 1024 1
timeout 300 python tools/tcompact.py c2 32
} > gpurun_out/r2/svd_$T.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2/svd_launch_$T.csv python tools/tcompact.py c2 1 > /dev/null 2>&1
