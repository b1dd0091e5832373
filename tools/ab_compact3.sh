python tools/tcompact.py c2 4 > gpurun_out/cmp_time.txt 2>&1
KVP_SVD_SPLIT=0 python tools/tcompact.py c2 4 > gpurun_out/cmp_time0.txt 2>&1
python tools/tcompact.py c2 4 >> gpurun_out/cmp_time.txt 2>&1
python tools/tcompact.py c2 32 >> gpurun_out/cmp_time.txt 2>&1
