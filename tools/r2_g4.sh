#!/bin/bash
# Round-2 late checkpoint: round script + the C5 two-tier sweep (r1 in {.125,.25,.375,.5} vs untiered).
T=$1
mkdir -p gpurun_out/r2
bash tools/r2_round.sh $T
for r in 0 0.125 0.25 0.375 0.5; do
  timeout 120 python tools/kbench_fused.py --config c5 --tier $r >> gpurun_out/r2/tier_sweep_$T.txt 2>&1
done
