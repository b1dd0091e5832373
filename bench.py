"""Benchmark: decode tokens/s over the compressed KV cache on B200.

Workload (BASELINE.json configs[1]): LLaVA-1.5-7B-shaped,
32 layers x 32 heads x 128 dim, 4 images x 576 visual tokens + 64 text tokens
per instance, batch 16 per GPU, visual K/V factored at rank 368 (4.0x),
textual tail dense and growing one token per decode step, bf16 cache, synthetic
data (Philox workload generator of the reference harness, random weights).

A step = one decode step for every instance through every layer (projection
GEMMs, tail append, compressed-cache attention + importance EMA, output GEMM),
i.e. the reference's decode_step (decoder.cpp:555-617) for all (instance,
layer) pairs.  The timed region covers the configuration's whole decode run
(256 steps: the textual tail grows from 64 to 320 rows) from the post-prefill
state; warm-up steps run first and the engine is reset to that state.
`value` times the steps with inputs resident in HBM; `e2e` times the same
steps through the host-buffer C-ABI call (kvp_engine_step_host: H2D of the
inputs, D2H of the outputs every step).  Per-step data (~10 GB) is far larger
than L2 (126 MB), so no explicit flush is needed.

Multi-GPU: one process per GPU.  `--gpus N` without a torchrun environment
re-launches itself under torch.distributed.run (127.0.0.1).  Instances are
split contiguously over ranks (paper_2603_23914_b200/shard.py): weak scaling
by default (the config's batch per GPU), strong scaling with --global-batch
(e.g. C3: 64 instances over 8 GPUs = 8 per GPU).  No collective on the
per-step path; the timed region is bracketed by barriers and reduced as the
max over ranks; final outputs are gathered to rank 0 once (NCCL).

--impl reference runs the reference's own CPU decode step (oracle/_ref) on the
host cores for the same config and metric (bounded sample, extrapolated).
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: geometry (H, Hkv, D), layers, batch per GPU, visual, textual, steps, rank
    "c2": dict(desc="LLaVA-1.5-7B all 32 layers, 4 images x 576 tokens + 64 text, batch 16/GPU, 4x compression",
               geom=(32, 32, 128), layers=32, batch=16, visual=2304, textual=64, steps=256, rank=368),
    "c3": dict(desc="LLaVA-1.5-13B 40 layers, 16 images x 256 tokens + 64 text, batch 64 (global), 8x compression",
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


def cpu_model():
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


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


def relaunch_under_torchrun(n):
    """`--gpus N` from a plain `python bench.py`: one process per GPU via
    torch.distributed.run on 127.0.0.1 (the driver's own launch form)."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


def dist_setup():
    """One process per GPU under torchrun: NCCL on a GPU box, gloo when no GPU is
    visible (the multi-process CPU tests)."""
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
    """Whole-job tokens/s when every rank decodes `batch_per_rank` instances."""
    return world * batch_per_rank * steps / (ms * 1e-3)


def shard_plan(cfg, world, rank, global_batch=None):
    """(global batch, this rank's [lo, hi) instance slice, scaling kind)."""
    from paper_2603_23914_b200.shard import instance_range
    if global_batch is None:
        gb = cfg["batch"] * world
        scaling = "weak"
    else:
        gb = global_batch
        scaling = "strong"
    lo, hi = instance_range(gb, world, rank)
    return gb, lo, hi, scaling


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
    desc = (f"{threads} (instance, layer) caches of the {cfg['geom']} geometry, one reference decode_step<float> "
            f"each in parallel per timed step ({steps} steps, median {pair_s:.2f} s); extrapolated linearly to "
            f"{cfg['batch']}x{cfg['layers']} pairs per decode step; CPU: {cpu_model()}")
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


def compaction_block(cfg, info, batch):
    """Prefill compaction against the tensor roofline: algorithmic flops
    2*T*W*k*(2q+2) per matrix, 2 matrices per (instance, layer)."""
    H, Hkv, D = cfg["geom"]
    T, W, R = cfg["visual"], Hkv * D, cfg["rank"]
    k = min(R + 8, min(T, W))
    flops = 2.0 * T * W * k * (2 * 2 + 2) * 2 * batch * cfg["layers"]
    peak, src = 1590.0, "fallback (B200_PROFILING.md)"
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        if d.get("bf16_tflops_sustained"):
            peak, src = float(d["bf16_tflops_sustained"]), "MEASURED_PEAKS.json bf16_tflops_sustained"
    achieved = flops / (info.compaction_ms * 1e-3) / 1e12
    return {"ms": info.compaction_ms, "matrices": 2 * batch * cfg["layers"], "shape": [T, W], "rank": R,
            "sketch": k, "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak if peak else None, "peak_source": src,
            "note": "randomized SVD + packing of every (instance, layer, K|V) visual segment on this rank, CUDA "
                    "events; the synthetic K/V generation is excluded; libraries warmed by one same-shape SVD"}


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed decode steps (default: the configuration's whole decode run, 256)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--global-batch", type=int, default=None,
                    help="split this many instances contiguously over the ranks (strong scaling); default: the "
                         "config's batch on every rank (weak scaling)")
    ap.add_argument("--factor-init", default="compaction", choices=["placeholder", "compaction"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--tier", type=float, nargs=2, default=None, metavar=("R1", "VALUE_FRACTION"),
                    help="two-tier values: first-group ratio and the second group's value-rank fraction "
                         "(default: the config's; 0 1 = untiered)")
    return ap.parse_args(argv)


def main():
    args = parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args.gpus))
    cfg = dict(CONFIGS[args.config])
    steps = args.steps if args.steps is not None else cfg["steps"]
    if args.tier is not None:
        cfg["tier"] = tuple(args.tier)
    tier = cfg.get("tier")
    if tier is not None and not (0.0 < tier[0] < 1.0 and tier[1] < 1.0):
        tier = None
    cfg["tier"] = tier
    world, rank, local = dist_setup()
    if args.config == "c3" and args.global_batch is None:
        args.global_batch = cfg["batch"]  # BASELINE: batch 64 sharded over the GPUs
    gb, lo, hi, scaling = shard_plan(cfg, world, rank, args.global_batch)
    B = hi - lo
    H, Hkv, D = cfg["geom"]
    config_block = {"workload": args.config, "description": cfg["desc"], "heads": H, "kv_heads": Hkv, "head_dim": D,
                    "layers": cfg["layers"], "global_batch": gb, "batch_per_gpu": B,
                    "visual_tokens": cfg["visual"], "textual_tokens": cfg["textual"], "rank": cfg["rank"],
                    "decode_steps_timed": steps, "tail_tokens_timed": [cfg["textual"] + 1, cfg["textual"] + steps],
                    "l2_flush": "not needed: per-step data (GBs) >> 126 MB L2",
                    "parallelism": f"instance-sharded x{world} ({scaling} scaling, no per-step collective; "
                                   f"one NCCL gather of outputs at the end)"}
    if tier is not None:
        config_block["tiering"] = {"ratios": [tier[0], 1.0 - tier[0]], "key_rank_fractions": [1.0, 1.0],
                                   "value_rank_fractions": [1.0, tier[1]]}

    if args.impl == "reference":
        if rank != 0:
            return
        rsteps, warmup = max(1, min(steps, 3)), min(args.warmup, 1)
        value, threads, desc, pair_s = cpu_reference(cfg, rsteps, warmup)
        line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus, "steps": rsteps,
                "warmup": warmup, "ms_per_step": 1e3 * cfg["batch"] / value, "higher_is_better": True,
                "scaling": scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic", "impl": "reference",
                "config": config_block,
                "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "reference",
                                 "sample": desc},
                "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    if not torch.cuda.is_available():
        raise SystemExit("bench.py --impl b200 needs a CUDA device (the product path has no CPU fallback)")
    from paper_2603_23914_b200 import _capi
    from paper_2603_23914_b200.engine import Engine, EngineSpec, ProfileSpec
    from paper_2603_23914_b200.shard import gather_instances

    torch.cuda.set_device(local)
    spec = EngineSpec(heads=H, kv_heads=Hkv, head_dim=D, layers=cfg["layers"], batch=B,
                      visual_tokens=cfg["visual"], textual_tokens=cfg["textual"],
                      decode_steps=max(steps, args.warmup), rank_k=cfg["rank"], rank_v=cfg["rank"],
                      visual=ProfileSpec(2 * cfg["rank"], cfg["rank"], 0.98, 1e-2), seed=0,
                      instance_offset=lo, factor_init=args.factor_init,
                      tier_ratio=tier[0] if tier else 0.0, tier_value_fraction=tier[1] if tier else 1.0)
    if args.factor_init == "compaction":
        warm_libraries(cfg)
    eng = Engine(spec)
    eng.prefill()
    info = eng.info()
    HD = H * D
    # decode inputs per global instance (harness.cpp:169-170: N(0,1)), this rank's slice
    gen = torch.Generator(device="cpu").manual_seed(1234)
    xs_all = torch.randn((steps, gb, HD), generator=gen, dtype=torch.float32)
    xs = xs_all[:, lo:hi].contiguous().cuda()
    ys = torch.empty((B, HD), device="cuda", dtype=torch.float32)
    stream = torch.cuda.current_stream()

    def run_steps(n):
        for t in range(n):
            eng.step(xs[t].data_ptr(), ys.data_ptr(), stream.cuda_stream)

    # ---- warm-up, then back to the post-prefill state
    run_steps(args.warmup)
    torch.cuda.synchronize()
    eng.reset_steps()
    # ---- attention alone at the first decode step's tail (roofline at both ends of the run)
    att_ms0, att_bytes0 = eng.time_attention(iters=3)
    eng.reset_steps()

    # ---- device-resident timing of the whole decode run
    sampler = ClockSampler(local)
    sampler.start()
    sampler.wait_first()
    barrier(world)
    torch.cuda.synchronize()
    launches0 = _capi.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    run_steps(steps)
    e1.record(stream)
    torch.cuda.synchronize()
    launches = _capi.launch_count() - launches0
    clocks = sampler.stop()
    barrier(world)
    ms = max_over_ranks(e0.elapsed_time(e1), world)
    value = gb * steps / (ms * 1e-3)
    # ---- once per run: final-step outputs of every instance to rank 0 (ordered merge, harness.cpp:400-412)
    gathered = gather_instances(ys, world, gb)

    # ---- roofline: the attention launches alone at the final tail length
    att_ms1, att_bytes1 = eng.time_attention(iters=3)
    peak, peak_src = load_peaks()
    achieved = att_bytes1 / (att_ms1 * 1e-3) / 1e9
    # DRAM bytes per layer from the committed ncu capture, only when it was taken at this run's final tail
    traffic = None
    ncu_file = ROOT / "profiles" / f"ncu_attention_{args.config}.json"
    if ncu_file.exists():
        nj = json.loads(ncu_file.read_text())
        if nj.get("tail_tokens") == cfg["textual"] + steps and nj.get("batch", B) == B:
            traffic = nj.get("dram_bytes_per_layer")
    # cache path (attention + EMA launches of every layer) at the mean of the run's first and last tail
    cache_ms_step = 0.5 * (att_ms0 + att_ms1) * cfg["layers"]
    cache_path = max_over_ranks(cache_ms_step, world)

    # ---- e2e through the host-buffer C-ABI call, same steps from the same state
    eng.reset_steps()
    xh = torch.empty((steps, B, HD), dtype=torch.float32, pin_memory=True)
    xh.copy_(xs_all[:, lo:hi])
    yh = torch.empty((B, HD), dtype=torch.float32, pin_memory=True)
    barrier(world)
    t0 = time.perf_counter()
    for t in range(steps):
        eng.step_host(xh[t].data_ptr(), yh.data_ptr())
    e2e_s = max_over_ranks(time.perf_counter() - t0, world)
    e2e_value = gb * steps / e2e_s

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            v, threads, desc, _ = cpu_reference(cfg, steps=1, warmup=0)
            cpu = {"value": v, "unit": "tokens/s", "cores": threads, "kind": "reference", "sample": desc}
        except Exception as exc:  # the oracle library is absent on this box
            cpu = {"value": None, "unit": "tokens/s", "cores": 0, "kind": "reference", "sample": f"unavailable: {exc}"}

    if rank == 0:
        out = gathered.double().cpu()
        line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": steps,
                "warmup": args.warmup, "ms_per_step": ms / steps, "higher_is_better": True, "scaling": scaling,
                "vs_baseline": None, "dtype": "bf16", "data": "synthetic (Philox workload generator, random weights)",
                "config": config_block,
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                             "frac": achieved / peak, "traffic": traffic,
                             "kernel": "decode attention (qdots + cluster core + vsum) per layer, final tail",
                             "peak_source": peak_src, "tail_tokens": cfg["textual"] + steps,
                             "ms_per_layer": att_ms1, "algorithmic_bytes_per_layer": att_bytes1,
                             "first_step": {"ms_per_layer": att_ms0, "algorithmic_bytes_per_layer": att_bytes0,
                                            "frac": att_bytes0 / (att_ms0 * 1e-3) / 1e9 / peak}},
                "cache_path": {"value": gb / (cache_path * 1e-3), "unit": "tokens/s",
                               "note": "attention + importance launches of every layer alone (no projections), "
                                       "mean of the first and last step's tail"},
                "cpu_baseline": cpu,
                "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": B * HD * 4,
                        "d2h_bytes_per_step": B * HD * 4},
                "gpu_launches": int(launches),
                "clocks": clocks,
                "gathered": {"instances": int(out.shape[0]), "output_l2": float(out.norm()),
                             "output_sum": float(out.sum())},
                "compaction_ms": info.compaction_ms if args.factor_init == "compaction" else None,
                "compaction": compaction_block(cfg, info, B) if args.factor_init == "compaction" else None,
                "factor_init": args.factor_init,
                "cluster": info.cluster}
        print(json.dumps(line), flush=True)
    eng.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
