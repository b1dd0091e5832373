"""Engine at a bench config, decode to the bench's final tail, then one attention-only replay
inside cudaProfilerStart/Stop, so `ncu --profile-from-start off` captures qdots/core/vsum of every
layer at that tail (the same state bench.py's roofline.achieved is timed at).

usage: ncu --profile-from-start off ... python tools/ncu_tail.py [config] [steps]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from bench import CONFIGS  # noqa: E402
from paper_2603_23914_b200.engine import Engine, EngineSpec, ProfileSpec  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 256
cfg = CONFIGS[name]
H, Hkv, D = cfg["geom"]
B = cfg["batch"]
spec = EngineSpec(heads=H, kv_heads=Hkv, head_dim=D, layers=cfg["layers"], batch=B, visual_tokens=cfg["visual"],
                  textual_tokens=cfg["textual"], decode_steps=steps, rank_k=cfg["rank"], rank_v=cfg["rank"],
                  visual=ProfileSpec(2 * cfg["rank"], cfg["rank"], 0.98, 1e-2), seed=0, factor_init="placeholder")
eng = Engine(spec)
eng.prefill()
x = torch.randn((B, H * D), device="cuda")
y = torch.empty_like(x)
for _ in range(steps):
    eng.step(x.data_ptr(), y.data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
ms, by = eng.time_attention(iters=1)
torch.cuda.synchronize()
torch.cuda.profiler.start()
ms, by = eng.time_attention(iters=1)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"tail {cfg['textual'] + steps} attention ms/layer {ms:.4f} algorithmic bytes/layer {by:.0f}")
