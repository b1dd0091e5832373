"""Benchmark: decode tokens/s over the compressed KV cache on B200.

Workload (BASELINE.json configs[1]): LLaVA-1.5-7B-shaped,
32 layers x 32 heads x 128 dim, 4 images x 576 visual tokens + 64 text tokens
per instance, batch 16 per GPU, visual K/V factored at rank 368 (4.0x),
textual tail dense and growing one token per decode step, bf16 cache, synthetic
data (Philox workload generator of the reference harness, random weights).

A step = one decode step for every instance through every layer (projection
GEMMs, tail append, compressed-cache attention + importance EMA, output GEMM),
i.e. the reference's decode_step (decoder.cpp:555-617) for all (instance,
layer) pairs.  `value` times steps with inputs resident in HBM; `e2e` times the
same steps through the host-buffer C-ABI call (kvp_engine_step_host: H2D of
the inputs, D2H of the outputs every step).  Per-step data (~10 GB) is far
larger than L2 (126 MB), so no explicit flush is needed.

Multi-GPU: one process per GPU (torchrun), every rank runs its own batch of
instances (weak scaling, no collective on the data path); the timed region is
bracketed by barriers, max over ranks.

--impl reference runs the reference's own CPU decode step (oracle/_ref) on the
host cores for the same config and metric (bounded sample, extrapolated).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: geometry (H, Hkv, D), layers, batch, visual, textual, steps, rank
    "c2": dict(desc="LLaVA-1.5-7B all 32 layers, 4 images x 576 tokens + 64 text, batch 16/GPU, 4x compression",
               geom=(32, 32, 128), layers=32, batch=16, visual=2304, textual=64, steps=256, rank=368),
    "c3": dict(desc="LLaVA-1.5-13B 40 layers, 16 images x 256 tokens + 64 text, batch 64/GPU, 8x compression",
               geom=(40, 40, 128), layers=40, batch=64, visual=4096, textual=64, steps=256, rank=284),
    "c5": dict(desc="VideoLLaVA-7B 8 frames x 256 tokens + 64 text, batch 32/GPU, rank 128, attention-aware "
                    "decompression: top 25% of tokens by importance at full rank, the rest at 1/4 of the value rank",
               geom=(32, 32, 128), layers=32, batch=32, visual=2048, textual=64, steps=256, rank=128,
               tier=(0.25, 0.25)),
    "c4_8x": dict(desc="Qwen-VL-7B-shaped 16 images x 256 tokens + 64 text, batch 16/GPU, 8x compression",
                  geom=(32, 32, 128), layers=32, batch=16, visual=4096, textual=64, steps=256, rank=256),
    "c4_4x": dict(desc="Qwen-VL-7B-shaped 16 images x 256 tokens + 64 text, batch 16/GPU, 4x compression",
                  geom=(32, 32, 128), layers=32, batch=16, visual=4096, textual=64, steps=256, rank=512),
    "c4_2x": dict(desc="Qwen-VL-7B-shaped 16 images x 256 tokens + 64 text, batch 16/GPU, 2x compression",
                  geom=(32, 32, 128), layers=32, batch=16, visual=4096, textual=64, steps=256, rank=1024),
}
METRIC = "decode tokens/sec over compressed KV-cache"


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        if d.get("hbm_gbs"):
            return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    return 6650.0, "fallback (B200_PROFILING.md; MEASURED_PEAKS.json absent)"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None
        self.th = None

    def start(self):
        q = "clocks.sm,clocks.max.sm,clocks_event_reasons.active"
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.th = threading.Thread(target=self._read, daemon=True)
        self.th.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 3:
                try:
                    self.samples.append((float(parts[0]), float(parts[1]), int(parts[2], 16), time.monotonic()))
                except ValueError:
                    pass

    def wait_first(self, timeout=5.0):
        """Block until nvidia-smi delivers its first sample (it needs ~0.1-0.5 s to start),
        so that the timed region that follows is covered."""
        end = time.monotonic() + timeout
        while self.proc and not self.samples and time.monotonic() < end:
            time.sleep(0.01)
        self.t_begin = time.monotonic()

    def stop(self):
        # one more sample after the timed region (100 ms period), so a short region is bracketed
        t_end = time.monotonic()
        end = t_end + 0.5
        while self.proc and not any(x[3] >= t_end for x in self.samples) and time.monotonic() < end:
            time.sleep(0.01)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.th:
            self.th.join(timeout=5)
        names = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
                 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        t0 = getattr(self, "t_begin", 0.0)
        # the samples that bracket the timed region: from the last one before it through the first one after
        before = [x for x in self.samples if x[3] < t0]
        window = ([before[-1]] if before else []) + [x for x in self.samples if x[3] >= t0]
        self.samples = window or self.samples
        sm = sorted(s[0] for s in self.samples)
        reasons = set()
        for _, _, r, _ in self.samples:
            for bit, n in names.items():
                if r & bit and n != "gpu_idle":
                    reasons.add(n)
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(s[1] for s in self.samples), "reasons": sorted(reasons)}


def dist_setup():
    """One process per GPU under torchrun: NCCL on a GPU box, gloo when no GPU is
    visible (the multi-process CPU tests).  Only the barrier and the max-over-ranks
    of the device-timed region use it: instances are sharded, no data-path collective."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        import torch
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_throughput(world, batch_per_rank, steps, ms):
    """Whole-job tokens/s: every rank decodes its own instances (weak scaling)."""
    return world * batch_per_rank * steps / (ms * 1e-3)


def cpu_reference(cfg, steps, warmup, threads=None):
    """Reference CPU decode step on a bounded sample (oracle/_ref)."""
    from oracle import cpu_baseline as cb
    threads = threads or cb.host_threads()
    tier = cfg.get("tier")
    tiering = (((tier[0], 1.0 - tier[0]), (1.0, 1.0), (1.0, tier[1])) if tier else None)
    sample = cb.ReferenceSample(cfg["geom"], cfg["visual"], cfg["textual"], cfg["rank"], cfg["rank"], threads,
                                tiering=tiering)
    for _ in range(warmup):
        sample.step()
    secs = [sample.step() for _ in range(steps)]
    pair_s = sorted(secs)[len(secs) // 2]
    value = cb.tokens_per_second(pair_s, cfg["batch"], cfg["layers"], threads)
    desc = (f"{threads} (instance, layer) caches of the {cfg['geom']} geometry, one reference decode_step each "
            f"in parallel per timed step ({steps} steps, median {pair_s:.2f} s); extrapolated to "
            f"{cfg['batch']}x{cfg['layers']} pairs per decode step")
    return value, threads, desc, pair_s


def warm_libraries(cfg):
    """One same-shape randomized SVD through kvp_truncated_svd before the
    engine's timed prefill, so the cuBLAS/cuSOLVER modules are paged in and
    loaded outside the compaction timing (a fresh box otherwise pays that on
    the first layer)."""
    import torch
    from paper_2603_23914_b200 import _capi

    H, Hkv, D = cfg["geom"]
    T, W, R = cfg["visual"], Hkv * D, cfg["rank"]
    a = torch.randn((2, T, W), device="cuda", dtype=torch.float32)
    left = torch.empty((2, T, R), device="cuda", dtype=torch.float32)
    right = torch.empty((2, R, W), device="cuda", dtype=torch.float32)
    _capi.call("kvp_truncated_svd", a.data_ptr(), 2, T, W, R, 1, 7, 8, 2, left.data_ptr(), right.data_ptr(),
               None, None)
    torch.cuda.synchronize()


def compaction_block(cfg, info, world):
    """Prefill compaction against the tensor roofline: algorithmic flops
    2*T*W*k*(2q+2) per matrix, 2 matrices per (instance, layer)."""
    H, Hkv, D = cfg["geom"]
    T, W, R = cfg["visual"], Hkv * D, cfg["rank"]
    k = min(R + 8, min(T, W))
    flops = 2.0 * T * W * k * (2 * 2 + 2) * 2 * cfg["batch"] * cfg["layers"]
    peak, src = 1590.0, "fallback (B200_PROFILING.md)"
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        if d.get("bf16_tflops_sustained"):
            peak, src = float(d["bf16_tflops_sustained"]), "MEASURED_PEAKS.json bf16_tflops_sustained"
    achieved = flops / (info.compaction_ms * 1e-3) / 1e12
    return {"ms": info.compaction_ms, "matrices": 2 * cfg["batch"] * cfg["layers"], "shape": [T, W], "rank": R,
            "sketch": k, "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak if peak else None, "peak_source": src,
            "note": "randomized SVD + packing of every (instance, layer, K|V) visual segment, CUDA events; "
                    "the synthetic K/V generation is excluded; cuBLAS/cuSOLVER warmed by one same-shape SVD beforehand"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--factor-init", default="compaction", choices=["placeholder", "compaction"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--tier", type=float, nargs=2, default=None, metavar=("R1", "VALUE_FRACTION"),
                    help="two-tier values: first-group ratio and the second group's value-rank fraction "
                         "(default: the config's; 0 1 = untiered)")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.tier is not None:
        cfg["tier"] = tuple(args.tier)
    tier = cfg.get("tier")
    if tier is not None and not (0.0 < tier[0] < 1.0 and tier[1] < 1.0):
        tier = None
    cfg["tier"] = tier
    world, rank, local = dist_setup()
    H, Hkv, D = cfg["geom"]
    config_block = {"workload": args.config, "description": cfg["desc"], "heads": H, "kv_heads": Hkv, "head_dim": D,
                    "layers": cfg["layers"], "batch_per_gpu": cfg["batch"], "global_batch": cfg["batch"] * world,
                    "visual_tokens": cfg["visual"], "textual_tokens": cfg["textual"], "rank": cfg["rank"],
                    "tail_tokens_at_timing": None, "l2_flush": "not needed: per-step data >> 126 MB L2",
                    "parallelism": f"instance-sharded x{world} (no data-path collective)"}
    if tier is not None:
        config_block["tiering"] = {"ratios": [tier[0], 1.0 - tier[0]], "key_rank_fractions": [1.0, 1.0],
                                   "value_rank_fractions": [1.0, tier[1]]}

    if args.impl == "reference":
        if rank != 0:
            return
        steps, warmup = max(1, min(args.steps, 3)), min(args.warmup, 1)
        value, threads, desc, pair_s = cpu_reference(cfg, steps, warmup)
        line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus, "steps": steps,
                "warmup": warmup, "ms_per_step": 1e3 * cfg["batch"] / value, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic", "impl": "reference",
                "config": config_block,
                "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "reference",
                                 "sample": desc},
                "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    from paper_2603_23914_b200 import _capi
    from paper_2603_23914_b200.engine import Engine, EngineSpec, ProfileSpec

    torch.cuda.set_device(local)
    total_steps = args.warmup + args.steps
    spec = EngineSpec(heads=H, kv_heads=Hkv, head_dim=D, layers=cfg["layers"], batch=cfg["batch"],
                      visual_tokens=cfg["visual"], textual_tokens=cfg["textual"],
                      decode_steps=max(cfg["steps"], total_steps), rank_k=cfg["rank"], rank_v=cfg["rank"],
                      visual=ProfileSpec(2 * cfg["rank"], cfg["rank"], 0.98, 1e-2), seed=rank,
                      factor_init=args.factor_init,
                      tier_ratio=tier[0] if tier else 0.0, tier_value_fraction=tier[1] if tier else 1.0)
    if args.factor_init == "compaction":
        warm_libraries(cfg)
    eng = Engine(spec)
    eng.prefill()
    info = eng.info()
    B, HD = cfg["batch"], H * D
    gen = torch.Generator(device="cuda").manual_seed(1234 + rank)
    xs = torch.randn((total_steps, B, HD), device="cuda", generator=gen, dtype=torch.float32)
    ys = torch.empty((B, HD), device="cuda", dtype=torch.float32)
    stream = torch.cuda.current_stream()

    def run_steps(lo, hi):
        for t in range(lo, hi):
            eng.step(xs[t].data_ptr(), ys.data_ptr(), stream.cuda_stream)

    # ---- device-resident timing
    run_steps(0, args.warmup)
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    sampler.wait_first()
    barrier(world)
    torch.cuda.synchronize()
    launches0 = _capi.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    run_steps(args.warmup, total_steps)
    e1.record(stream)
    torch.cuda.synchronize()
    launches = _capi.launch_count() - launches0
    clocks = sampler.stop()
    barrier(world)
    ms = max_over_ranks(e0.elapsed_time(e1), world)
    tail_at = cfg["textual"] + args.warmup + 1
    config_block["tail_tokens_at_timing"] = [tail_at, tail_at + args.steps - 1]
    value = aggregate_throughput(world, B, args.steps, ms)

    # ---- roofline: the attention launches alone at the final tail length
    att_ms, att_bytes = eng.time_attention(iters=3)
    peak, peak_src = load_peaks()
    achieved = att_bytes / (att_ms * 1e-3) / 1e9
    traffic = None
    ncu_file = ROOT / "profiles" / f"ncu_attention_{args.config}.json"
    if ncu_file.exists():
        traffic = json.loads(ncu_file.read_text()).get("dram_bytes_per_layer")

    # ---- e2e through the host-buffer C-ABI call
    eng.reset_steps()
    xh = torch.empty((total_steps, B, HD), dtype=torch.float32, pin_memory=True)
    xh.copy_(xs.cpu())
    yh = torch.empty((B, HD), dtype=torch.float32, pin_memory=True)
    for t in range(args.warmup):
        eng.step_host(xh[t].data_ptr(), yh.data_ptr())
    barrier(world)
    t0 = time.perf_counter()
    for t in range(args.warmup, total_steps):
        eng.step_host(xh[t].data_ptr(), yh.data_ptr())
    e2e_s = max_over_ranks(time.perf_counter() - t0, world)
    e2e_value = world * B * args.steps / e2e_s

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            v, threads, desc, _ = cpu_reference(cfg, steps=1, warmup=0)
            cpu = {"value": v, "unit": "tokens/s", "cores": threads, "kind": "reference", "sample": desc}
        except Exception as exc:  # the oracle library is absent on this box
            cpu = {"value": None, "unit": "tokens/s", "cores": 0, "kind": "reference", "sample": f"unavailable: {exc}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "bf16", "data": "synthetic (Philox workload generator, random weights)",
                "config": config_block,
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                             "frac": achieved / peak, "traffic": traffic,
                             "kernel": "decode attention (qdots + cluster core + vsum) per layer",
                             "peak_source": peak_src,
                             "ms_per_layer": att_ms, "algorithmic_bytes_per_layer": att_bytes},
                "cpu_baseline": cpu,
                "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": B * HD * 4,
                        "d2h_bytes_per_step": B * HD * 4},
                "gpu_launches": int(launches),
                "clocks": clocks,
                "compaction_ms": info.compaction_ms if args.factor_init == "compaction" else None,
                "compaction": compaction_block(cfg, info, world) if args.factor_init == "compaction" else None,
                "factor_init": args.factor_init,
                "cluster": info.cluster}
        print(json.dumps(line), flush=True)
    eng.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
