#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2/team6_$1.txt
for d in 0 1; do echo "== dbg $d" >> $O; KVP_TEAM_DBG=$d timeout 120 python tools/kbench_fused.py --config c2 --cluster 0 --trace >> $O 2>&1; done
for cfg in c2 c5 c4_8x c4_2x; do echo "== $cfg" >> $O; timeout 120 python tools/kbench_fused.py --config $cfg --cluster 0 >> $O 2>&1; done
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_parity_configs.py tests/test_gpu_engine.py -x -q >> $O 2>&1
