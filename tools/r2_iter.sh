#!/bin/bash
# One iteration on the fused decode kernel: parity of the fused path, kernel timing + phase trace, short bench.
tag=${1:-x}
mkdir -p gpurun_out/p
timeout 600 python -m pytest tests/test_gpu_fused.py tests/test_gpu_parity_configs.py -x -q -k "fused" > gpurun_out/p/par_$tag.txt 2>&1
tail -3 gpurun_out/p/par_$tag.txt
for cfg in c2 c3 c5; do
  echo "== $cfg" >> gpurun_out/p/kb_$tag.txt
  timeout 120 python tools/kbench_fused.py --config $cfg --trace >> gpurun_out/p/kb_$tag.txt 2>&1
done
grep frac gpurun_out/p/kb_$tag.txt
if [ "$2" = "bench" ]; then timeout 400 python bench.py > gpurun_out/p/bench_$tag.json 2> gpurun_out/p/bench_$tag.err; cat gpurun_out/p/bench_$tag.json | head -c 600; fi
