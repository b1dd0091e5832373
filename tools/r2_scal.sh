#!/bin/bash
# Per-kernel serialised durations of qdots / core / vsum vs batch (fixed cost + per-byte cost).
mkdir -p gpurun_out/p
for b in 16 8 4; do
  KVP_SPLIT_SMS=$((9*b)) timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/p/scal_b$b.csv python tools/kbench_fused.py --config c2 --batch $b --layers 2 --iters 1 > /dev/null 2>&1
done
for b in 16 8 4; do echo "== B=$b"; python - <<PY
import csv,collections
d=collections.defaultdict(list)
for r in csv.DictReader(l for l in open("gpurun_out/p/scal_b$b.csv") if l.startswith('"')):
    if r["Metric Name"]=="gpu__time_duration.sum": d[r["Kernel Name"][:40]].append(float(r["Metric Value"]))
for k,v in d.items(): print(f"{k:42s} n={len(v)} median={sorted(v)[len(v)//2]:.0f} ns")
PY
done
