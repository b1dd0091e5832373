"""Microbenchmark of the fused decode kernel alone (kvp_decode_fused), per
layer launch, rotating over several layers' caches so the working set is far
larger than L2.  Prints achieved algorithmic GB/s vs MEASURED_PEAKS.json."""
import argparse
import ctypes as C
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from paper_2603_23914_b200 import _capi as capi  # noqa: E402
from paper_2603_23914_b200._capi import FusedDesc  # noqa: E402

CONFIGS = {
    "c2": dict(B=16, H=32, Hkv=32, D=128, n=2304, rk=368, rv=368, nt=64 + 128, cap=320),
    "c3": dict(B=64, H=40, Hkv=40, D=128, n=4096, rk=284, rv=284, nt=64 + 128, cap=320),
    "c5": dict(B=32, H=32, Hkv=32, D=128, n=2048, rk=128, rv=128, nt=64 + 128, cap=320),
    "c4_8x": dict(B=16, H=32, Hkv=32, D=128, n=4096, rk=256, rv=256, nt=64 + 128, cap=320),
    "c4_2x": dict(B=16, H=32, Hkv=32, D=128, n=4096, rk=1024, rv=1024, nt=64 + 128, cap=320),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--cluster", type=int, default=0)
    ap.add_argument("--trace", action="store_true")
    ap.add_argument("--ld", type=int, default=0)
    ap.add_argument("--batch", type=int, default=0, help="override the config's batch")
    ap.add_argument("--streams", type=int, default=1, help="layers round-robin over this many streams")
    ap.add_argument("--tier", type=float, default=0.0,
                    help="two-tier values: first-group ratio r1 (the rest use a quarter of the value rank)")
    args = ap.parse_args()
    c = CONFIGS[args.config]
    B, H, Hkv, D, n, rk, rv, nt, cap = (c[k] for k in ("B", "H", "Hkv", "D", "n", "rk", "rv", "nt", "cap"))
    B = args.batch or B
    W = Hkv * D
    ld = args.ld or (max(rk, rv) + 7) // 8 * 8
    dev = "cuda"
    bf = torch.bfloat16
    layers = []
    for _ in range(args.layers):
        def packed(r):
            src = torch.randn(B, n, r, device=dev).to(bf)
            out = torch.empty(capi.lib().kvp_packed_left_bytes(B, n, r), dtype=torch.uint8, device=dev)
            capi.call("kvp_pack_left", src.data_ptr(), r, B, n, r, out.data_ptr(), None)
            return out
        L = dict(lk=packed(rk), lv=packed(rv),
                 rk=(torch.randn(B, rk, W, device=dev) / W ** 0.5).to(bf),
                 rv=(torch.randn(B, rv, W, device=dev) / W ** 0.5).to(bf),
                 tk=torch.randn(B, cap, W, device=dev).to(bf), tv=torch.randn(B, cap, W, device=dev).to(bf),
                 q=torch.randn(B, H * D, device=dev), imp=torch.rand(B, n + cap, device=dev, dtype=torch.float64),
                 ctx=torch.empty(B, H * D, device=dev, dtype=bf))
        L["desc"] = FusedDesc(H, Hkv, D, B, n, rk, rv, 0, cap, nt, None, args.cluster, 1, L["lk"].data_ptr(),
                              L["rk"].data_ptr(), L["lv"].data_ptr(), L["rv"].data_ptr(), L["tk"].data_ptr(),
                              L["tv"].data_ptr(), L["q"].data_ptr(), L["imp"].data_ptr(), n + cap, 0.25, None,
                              L["ctx"].data_ptr())
        if args.tier > 0:
            rv2 = max(1, min(rv - 1, int(0.25 * rv + 0.5)))
            L["tier"] = (torch.rand(B, n, device=dev) >= args.tier).to(torch.uint8)
            L["desc"].tier2_value_rank = rv2
            L["desc"].value_tier = L["tier"].data_ptr()
        layers.append(L)
    fn = capi.lib().kvp_decode_fused
    fn.argtypes = [C.POINTER(FusedDesc), C.c_void_p]
    capi.lib().kvp_decode_fused_workspace.argtypes = [C.POINTER(FusedDesc)]
    capi.lib().kvp_decode_fused_workspace.restype = C.c_size_t
    for L in layers:
        nbytes = capi.lib().kvp_decode_fused_workspace(C.byref(L["desc"]))
        L["ws"] = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
        L["desc"].workspace, L["desc"].workspace_bytes = L["ws"].data_ptr(), nbytes
    stream = torch.cuda.current_stream().cuda_stream
    for L in layers:  # warm-up
        capi.check(fn(C.byref(L["desc"]), stream))
    torch.cuda.synchronize()
    if args.trace:
        cl = max(args.cluster, 18)  # trace buffer sized for the largest CTA count per instance
        buf = torch.zeros(B * cl * 32, dtype=torch.int64, device=dev)
        capi.lib().kvp_debug_fused_trace.argtypes = [C.c_void_p]
        capi.lib().kvp_debug_fused_trace(buf.data_ptr())
        capi.check(fn(C.byref(layers[0]["desc"]), stream))
        torch.cuda.synchronize()
        capi.lib().kvp_debug_fused_trace(None)
        if args.cluster > 0:
            capi.lib().kvp_debug_fused_max_clusters.argtypes = [C.POINTER(FusedDesc)]
            print("max active clusters:", capi.lib().kvp_debug_fused_max_clusters(C.byref(layers[0]["desc"])))
        t = buf.view(B * cl, 32)[:, :19].double().cpu()
        t = t[t[:, 0] > 0]
        t0 = t[:, 0].min()
        names = ["start", "S ready", "local stats", "p tiles", "U ready", "end", "cluster stats", "mma U issued",
                 "mma P ok", "mma S done", "prod LV0", "mma p0 ok", "mma p1 ok", "mma p2 ok", "prod last", "EMA done",
                 "bar stats", "bar released", "bar passed"]
        rel = (t - t0) / 1000.0
        print("phase (us since first CTA start): median / max over CTAs")
        for k, n_ in enumerate(names):
            print(f"  {n_:10s} {rel[:, k].median().item():8.2f} {rel[:, k].max().item():8.2f}")
    # capture the layer launches once in a CUDA graph: the timed region is GPU work only
    g = torch.cuda.CUDAGraph()
    s_cap = torch.cuda.Stream()
    with torch.cuda.stream(s_cap):
        g.capture_begin()
        if args.streams > 1:
            side = [torch.cuda.Stream() for _ in range(args.streams)]
            ev0 = torch.cuda.Event()
            ev0.record(s_cap)
            for sd in side:
                sd.wait_event(ev0)
            for i, L in enumerate(layers):
                capi.check(fn(C.byref(L["desc"]), side[i % args.streams].cuda_stream))
            for sd in side:
                e = torch.cuda.Event()
                e.record(sd)
                s_cap.wait_event(e)
        else:
            for L in layers:
                capi.check(fn(C.byref(L["desc"]), s_cap.cuda_stream))
        g.capture_end()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(args.iters):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / (args.iters * len(layers))
    per_inst = 2 * (n * (rk + rv) + (rk + rv) * W + 2 * nt * W) + 16 * (n + nt) + H * D * 4 + H * D * 2
    gbs = B * per_inst / (ms * 1e-3) / 1e9
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = peaks.get("hbm_gbs", 6650.0)
    print(json.dumps(dict(config=args.config, tier_r1=args.tier, ms_per_layer=round(ms, 4), bytes_per_layer=B * per_inst,
                          achieved_gbs=round(gbs, 1), peak_gbs=peak, frac=round(gbs / peak, 3))))


if __name__ == "__main__":
    main()
