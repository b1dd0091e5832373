timeout 900 python -m pytest tests -m gpu -x -q -k "compaction or kvpack or svd" > gpurun_out/cmp_tests.txt 2>&1
python tools/check_compaction.py 2304 4096 368 3 > gpurun_out/cmp_acc.txt 2>&1
python tools/tcompact.py c2 4 > gpurun_out/cmp_time.txt 2>&1
