#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2/team_$1.txt
timeout 120 python tools/kbench_fused.py --config c2 --cluster 0 --iters 5 >> $O 2>&1 || echo "kbench c2 rc=$?" >> $O
timeout 600 python -m pytest tests/test_gpu_fused.py tests/test_gpu_parity_configs.py -x -q >> $O 2>&1
for cfg in c2 c3 c5 c4_8x c4_2x; do
  for t in 1 0; do
    echo "== $cfg team $t" >> $O
    KVP_TEAM=$t timeout 120 python tools/kbench_fused.py --config $cfg --cluster 0 >> $O 2>&1
  done
done
timeout 600 python -m pytest tests/test_gpu_engine.py tests/test_gpu_cache.py -x -q >> $O 2>&1
for t in 1 0; do echo "== bench team $t" >> $O; KVP_TEAM=$t timeout 300 python bench.py --steps 64 --no-cpu-baseline --factor-init placeholder 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['ms_per_layer'], d['roofline']['frac'], d['cache_path']['value'])" >> $O 2>&1; done
