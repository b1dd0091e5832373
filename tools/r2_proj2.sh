#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2/proj2_$1.txt
for d in 0 1 2 3; do echo "dbg $d" >> $O; KVP_PG_DBG=$d timeout 60 python tools/kbench_proj.py >> $O 2>&1; KVP_PG_DBG=$d timeout 60 python tools/kbench_proj.py --N 4096 >> $O 2>&1; done
for d in 0 3; do echo "dbg $d stages 4" >> $O; KVP_PG_STAGES=4 KVP_PG_DBG=$d timeout 60 python tools/kbench_proj.py >> $O 2>&1; done
