#!/bin/bash
# Other BASELINE configurations on one B200: decode + compaction (whole configured step count for decode is not
# needed here: 64 steps), plus C2 compaction accuracy tests.
mkdir -p gpurun_out/r2
T=$1
for cfg in c3 c4_8x c4_4x c4_2x c5; do
  timeout 900 python bench.py --config $cfg --steps 64 --no-cpu-baseline > gpurun_out/r2/cfg_${cfg}_$T.json 2> gpurun_out/r2/cfg_${cfg}_$T.err
done
