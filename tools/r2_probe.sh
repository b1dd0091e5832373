#!/bin/bash
# Fused decode timing + per-CTA phase trace (split mode) on one box.
mkdir -p gpurun_out/p
tag=${1:-x}
for cfg in c2 c3; do
  echo "== $cfg" >> gpurun_out/p/kb_$tag.txt
  timeout 120 python tools/kbench_fused.py --config $cfg --trace >> gpurun_out/p/kb_$tag.txt 2>&1
done
