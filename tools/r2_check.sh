#!/bin/bash
# GPU-box check: full -m gpu suite, smoke, one default bench line.
mkdir -p gpurun_out/r2
timeout 1500 python -m pytest tests -m gpu -q -rA -s > gpurun_out/r2/tests_$1.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2/smoke_$1.txt 2>&1
timeout 600 python bench.py > gpurun_out/r2/bench_$1.json 2> gpurun_out/r2/bench_$1.err
