timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/full_tests.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full_smoke.txt 2>&1
python bench.py > gpurun_out/full_bench.json 2> gpurun_out/full_bench.err
