#!/bin/bash
mkdir -p gpurun_out/r2
T=$1
{
timeout 600 python -m pytest tests/test_kvpack_api.py -k "rank_deficient or graded or matches_numpy or variance" -m gpu -q -s 2>&1 | tail -60
} > gpurun_out/r2/svd_$T.txt 2>&1
