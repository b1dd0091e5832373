import sys, time
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import torch
t0 = time.time(); torch.zeros(1).cuda(); print("torch init", time.time() - t0, flush=True)
from test_gpu_engine import make_engine
for i in range(2):
    t0 = time.time(); eng = make_engine(); print("prefill", time.time() - t0, eng.info().compaction_ms, flush=True)
    eng.close()
