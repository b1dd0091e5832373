B="python bench.py --no-cpu-baseline --factor-init placeholder --steps 30 --warmup 5"
timeout 600 python -m pytest tests -m gpu -x -q -k "fused or engine" > gpurun_out/pdl_tests.txt 2>&1
$B > gpurun_out/ab_pdl1.json 2> gpurun_out/ab_pdl1.err
KVP_PDL=0 $B > gpurun_out/ab_pdl0.json 2> gpurun_out/ab_pdl0.err
$B > gpurun_out/ab_pdl1b.json 2>&1
python tools/kbench_fused.py c2 > gpurun_out/kb_pdl1.txt 2>&1
KVP_PDL=0 python tools/kbench_fused.py c2 > gpurun_out/kb_pdl0.txt 2>&1
