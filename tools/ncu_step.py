"""Engine at a bench config, decode `steps` steps, then ONE whole decode step (all layers: projections,
attention, importance, tiers) inside cudaProfilerStart/Stop, so `ncu --profile-from-start off` gives the
step's launch list (per-kernel shares of one step).

usage: ncu --profile-from-start off --metrics gpu__time_duration.sum ... python tools/ncu_step.py [config] [steps]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from bench import CONFIGS  # noqa: E402
from paper_2603_23914_b200.engine import Engine, EngineSpec, ProfileSpec  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 128
cfg = CONFIGS[name]
H, Hkv, D = cfg["geom"]
B = cfg["batch"]
spec = EngineSpec(heads=H, kv_heads=Hkv, head_dim=D, layers=cfg["layers"], batch=B, visual_tokens=cfg["visual"],
                  textual_tokens=cfg["textual"], decode_steps=steps + 1, rank_k=cfg["rank"], rank_v=cfg["rank"],
                  visual=ProfileSpec(2 * cfg["rank"], cfg["rank"], 0.98, 1e-2), seed=0, factor_init="placeholder")
eng = Engine(spec)
eng.prefill()
x = torch.randn((B, H * D), device="cuda")
y = torch.empty_like(x)
for _ in range(steps):
    eng.step(x.data_ptr(), y.data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
torch.cuda.profiler.start()
eng.step(x.data_ptr(), y.data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"profiled decode step {steps + 1} (tail {cfg['textual'] + steps + 1})")
