#!/bin/bash
mkdir -p gpurun_out/r2
T=$1
{
timeout 900 python -m pytest tests/test_kvpack_api.py tests/test_snapshot.py tests/test_gpu_parity_configs.py tests/test_gpu_engine.py -k "quantize or snapshot or svd or singular or variance or compaction or device_cache or decodes" -m gpu -q -rfE 2>&1 | tail -8
timeout 300 python tools/check_compaction.py 2304 4096 368 1
timeout 600 python tools/tcompact.py c2 32 2
timeout 600 python tools/tcompact.py c3 4 2
} > gpurun_out/r2/check2_$T.txt 2>&1
