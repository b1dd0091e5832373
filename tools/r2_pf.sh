#!/bin/bash
# L2-prefetch A/B of the decode attention (KVP_PF bits), projection GEMM tests, engine bench A/B.
mkdir -p gpurun_out/r2
O=gpurun_out/r2/pf_$1.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv >> $O 2>&1
timeout 300 python -m pytest tests/test_gpu_proj.py tests/test_gpu_engine.py -x -q >> $O 2>&1
timeout 120 python tools/kbench_fused.py --config c2 --cluster 0 --trace >> $O 2>&1
for pf in 0 1 2 4 8 3 6 7 12 15 0; do
  echo "== c2 pf $pf" >> $O
  KVP_PF=$pf timeout 120 python tools/kbench_fused.py --config c2 --cluster 0 >> $O 2>&1
done
for pf in 0 15; do
  echo "== c3 pf $pf" >> $O
  KVP_PF=$pf timeout 120 python tools/kbench_fused.py --config c3 --cluster 0 >> $O 2>&1
done
for pf in 0 31; do
  echo "== bench pf $pf" >> $O
  KVP_PF=$pf timeout 300 python bench.py --steps 64 --no-cpu-baseline >> $O 2>>gpurun_out/r2/pf_$1.err
done
echo "== bench cublas" >> $O
KVP_PROJ=cublas timeout 300 python bench.py --steps 64 --no-cpu-baseline >> $O 2>>gpurun_out/r2/pf_$1.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"qdots|core|vsum" -c 24 --csv --log-file gpurun_out/r2/launch_$1.csv python tools/kbench_fused.py --config c2 --cluster 0 --iters 1 --layers 4 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2/launch_bench_$1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --factor-init placeholder > /dev/null 2>&1
