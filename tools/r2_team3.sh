#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2/team7_$1.txt
run() { timeout 300 python bench.py --steps 64 --no-cpu-baseline --factor-init placeholder 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['ms_per_layer'], d['roofline']['frac'], d['cache_path']['value'])" >> $O 2>&1; }
echo "== team" >> $O; run
echo "== team pf" >> $O; KVP_TEAM_DBG=4 run
echo "== noteam" >> $O; KVP_TEAM=0 run
echo "== team tc" >> $O; KVP_PROJ=tc run
echo "== team pf tc" >> $O; KVP_PROJ=tc KVP_TEAM_DBG=4 run
