python tools/check_compaction.py 2304 4096 368 2 > gpurun_out/cmp_acc_a.txt 2>&1
KVP_SVD_PASSES=2 python tools/check_compaction.py 2304 4096 368 2 > gpurun_out/cmp_acc_b.txt 2>&1
KVP_SVD_FP32=1 python tools/check_compaction.py 2304 4096 368 2 > gpurun_out/cmp_acc_c.txt 2>&1
KVP_SVD_FP32=1 KVP_SVD_PASSES=2 python tools/check_compaction.py 2304 4096 368 2 > gpurun_out/cmp_acc_d.txt 2>&1
