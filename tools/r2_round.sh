#!/bin/bash
# Round checkpoint: -m gpu suite, smoke, default bench (C2), compaction launch list (1 layer),
# attention ncu at the bench's final tail.
mkdir -p gpurun_out/r2
T=$1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2/gpu_$T.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rfE --timeout 600 > gpurun_out/r2/tests_$T.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2/smoke_$T.txt 2>&1
timeout 900 python bench.py > gpurun_out/r2/bench_$T.json 2> gpurun_out/r2/bench_$T.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2/compact_launch_$T.csv python tools/tcompact.py c2 1 > /dev/null 2>&1
bash tools/r2_prof_att.sh $T
