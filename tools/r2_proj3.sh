#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2/proj3_$1.txt
timeout 300 python -m pytest tests/test_gpu_proj.py -x -q >> $O 2>&1
for d in 0 3; do echo "dbg $d" >> $O; KVP_PG_DBG=$d timeout 60 python tools/kbench_proj.py --trace >> $O 2>&1; KVP_PG_DBG=$d timeout 60 python tools/kbench_proj.py --N 4096 --trace >> $O 2>&1; done
timeout 60 python tools/kbench_proj.py --B 64 --K 5120 --N 15360 >> $O 2>&1
timeout 60 python tools/kbench_proj.py --B 64 --K 5120 --N 5120 >> $O 2>&1
