#!/bin/bash
# Serialised per-kernel durations + DRAM bytes of the decode kernels (kbench, C2 B=16).
mkdir -p gpurun_out/p
tag=${1:-x}; cfg=${2:-c2}
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  -k regex:"qdots|core_k|vsum" --log-file gpurun_out/p/ncuk_$tag.csv python tools/kbench_fused.py --config $cfg --layers 2 --iters 1 > /dev/null 2>&1
python - <<PY
import csv,collections
d=collections.defaultdict(lambda: collections.defaultdict(list))
for r in csv.DictReader(l for l in open("gpurun_out/p/ncuk_$tag.csv") if l.startswith('"')):
    d[r["Kernel Name"][:36]][r["Metric Name"]].append(float(r["Metric Value"]))
for k,m in d.items():
    t=sorted(m["gpu__time_duration.sum"]); rb=sorted(m["dram__bytes_read.sum"]); 
    print(f"{k:38s} n={len(t)} t={t[len(t)//2]/1e3:.2f}us read={rb[len(rb)//2]/1e6:.1f}MB")
PY
