#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2/team9_$1.txt
timeout 120 python tools/kbench_fused.py --config c2 --cluster 0 --trace >> $O 2>&1
for cfg in c2 c5 c4_8x c4_2x; do for t in 1 0; do echo "== $cfg team $t" >> $O; KVP_TEAM=$t timeout 120 python tools/kbench_fused.py --config $cfg --cluster 0 >> $O 2>&1; done; done
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_parity_configs.py -x -q -k "fused" >> $O 2>&1
