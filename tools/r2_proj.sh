#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2/proj_$1.txt
timeout 300 python -m pytest tests/test_gpu_proj.py -x -q >> $O 2>&1
for shape in "16 4096 12288" "16 4096 4096" "64 5120 15360"; do
  set -- $shape
  timeout 60 python tools/kbench_proj.py --B $1 --K $2 --N $3 >> $O 2>&1
done
for st in 4 8; do echo "stages $st" >> $O; KVP_PG_STAGES=$st timeout 60 python tools/kbench_proj.py >> $O 2>&1; done
echo "nopdl" >> $O; KVP_PG_PDL=0 timeout 60 python tools/kbench_proj.py >> $O 2>&1
for gr in 74 96 128; do echo "grid $gr" >> $O; KVP_PG_GRID=$gr timeout 60 python tools/kbench_proj.py >> $O 2>&1; done
timeout 300 ncu --set full --clock-control none -k regex:proj_gemm -c 1 -o gpurun_out/r2/proj_full -f python tools/kbench_proj.py --iters 1 --copies 1 > /dev/null 2>&1
