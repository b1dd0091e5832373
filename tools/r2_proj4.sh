#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2/proj4_$1.txt
for st in 6 4 3; do echo "== stages $st" >> $O; KVP_PG_STAGES=$st timeout 300 python bench.py --steps 32 --no-cpu-baseline --factor-init placeholder 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['ms_per_layer'], d['cache_path']['value'])" >> $O 2>&1; done
echo "== cublas" >> $O; KVP_PROJ=cublas timeout 300 python bench.py --steps 32 --no-cpu-baseline --factor-init placeholder 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['ms_per_layer'], d['cache_path']['value'])" >> $O 2>&1
timeout 300 python -m pytest tests/test_gpu_engine.py -x -q >> $O 2>&1
