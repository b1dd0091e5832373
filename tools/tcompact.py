"""Time the engine's prefill compaction at a bench config with fewer layers.

usage: python tools/tcompact.py [config] [layers]
"""
import sys
import time

sys.path.insert(0, "/root/repo")
import torch  # noqa: E402

from bench import CONFIGS  # noqa: E402
from paper_2603_23914_b200.engine import Engine, EngineSpec  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
layers = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = CONFIGS[name]
H, Hkv, D = cfg["geom"]
torch.zeros(1).cuda()
for rep in range(int(sys.argv[3]) if len(sys.argv) > 3 else 2):
    spec = EngineSpec(heads=H, kv_heads=Hkv, head_dim=D, layers=layers, batch=cfg["batch"],
                      visual_tokens=cfg["visual"], textual_tokens=cfg["textual"], decode_steps=4,
                      rank_k=cfg["rank"], rank_v=cfg["rank"], factor_init="compaction")
    t0 = time.time()
    eng = Engine(spec)
    eng.prefill()
    print(f"{name} layers={layers} rep={rep} wall {time.time() - t0:.3f}s compaction_ms {eng.info().compaction_ms:.1f}",
          flush=True)
    eng.close()
