# Round-end: GPU tests, smoke, default bench, reference arm, decode launch list and attention capture
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/final_tests.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.txt 2>&1
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'qdots|core_kernel|vsum|nvjet|to_bf16|bump_counter|gemm' -c 3000 --csv --log-file gpurun_out/launches_decode.csv python bench.py --steps 3 --warmup 2 --no-cpu-baseline --factor-init placeholder > gpurun_out/prof1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'core_kernel|qdots|vsum' -s 30 -c 3 -o gpurun_out/attn_c2 -f python bench.py --steps 2 --warmup 1 --no-cpu-baseline --factor-init placeholder > gpurun_out/prof2.log 2>&1
