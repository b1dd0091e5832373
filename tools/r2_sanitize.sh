#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over small invocations of every hand-written kernel.
mkdir -p gpurun_out/r2
T=$1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_small.py > gpurun_out/r2/sanitize_${tool}_$T.txt 2>&1
done
