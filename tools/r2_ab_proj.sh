#!/bin/bash
# Projection GEMM A/B inside the whole decode step (C2, 256 steps, placeholder factors), then sanitizers.
mkdir -p gpurun_out/r2
T=$1
for rep in 1 2; do
for mode in cublas tc; do
  echo "== $mode rep $rep" >> gpurun_out/r2/abproj_$T.txt
  KVP_PROJ=$mode timeout 300 python bench.py --no-cpu-baseline --factor-init placeholder 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['ms_per_step'], d['roofline']['ms_per_layer'], d['cache_path']['value'])" >> gpurun_out/r2/abproj_$T.txt 2>&1
done
done
bash tools/r2_sanitize.sh $T
