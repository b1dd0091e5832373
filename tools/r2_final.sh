#!/bin/bash
# Final round check: GPU suite, smoke, default bench, compaction launch list, attention ncu at the
# final tail, sanitizers.
mkdir -p gpurun_out/r2
T=$1
bash tools/r2_round.sh $T
bash tools/r2_sanitize.sh $T
