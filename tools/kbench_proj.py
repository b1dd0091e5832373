"""Microbenchmark of the projection GEMM (kvp_matmul_packed) against torch.mm (cuBLAS) on the
decode step's shapes, rotating over several weight copies so the weights stream from HBM."""
import argparse
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2603_23914_b200 import _capi as capi  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--B", type=int, default=16)
    ap.add_argument("--K", type=int, default=4096)
    ap.add_argument("--N", type=int, default=12288)
    ap.add_argument("--copies", type=int, default=4)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--trace", action="store_true")
    a = ap.parse_args()
    B, K, N = a.B, a.K, a.N
    x = torch.randn(B, K, device="cuda").to(torch.bfloat16)
    ws_ = [(torch.randn(K, N, device="cuda") / K ** 0.5).to(torch.bfloat16) for _ in range(a.copies)]
    pks = []
    for w in ws_:
        pk = torch.empty(capi.lib().kvp_packed_weight_bytes(K, N), dtype=torch.uint8, device="cuda")
        capi.call("kvp_pack_weight", w.data_ptr(), K, N, pk.data_ptr(), None)
        pks.append(pk)
    wsp = torch.zeros(capi.lib().kvp_matmul_packed_workspace(K, N, B), dtype=torch.uint8, device="cuda")
    out = torch.empty(B, N, device="cuda")
    s = torch.cuda.Stream()

    def ours():
        for pk in pks:
            capi.call("kvp_matmul_packed", x.data_ptr(), B, K, pk.data_ptr(), N, out.data_ptr(), N, 0, wsp.data_ptr(),
                      s.cuda_stream)

    def lib():
        for w in ws_:
            torch.mm(x, w, out_dtype=torch.float32) if hasattr(torch, "_no_such") else torch.mm(x, w)

    res = {}
    for name, fn in (("ours", ours), ("cublas", lib)):
        with torch.cuda.stream(s):
            fn()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            g.capture_begin()
            fn()
            g.capture_end()
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.iters):
                g.replay()
            e1.record()
            torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (a.iters * a.copies)
        res[name] = dict(us=round(us, 2), gbs=round(2 * K * N / us / 1e3, 1))
    if a.trace:
        import ctypes as C
        buf = torch.zeros(2, 160 * 8, dtype=torch.int64, device="cuda")
        capi.lib().kvp_debug_proj_trace.argtypes = [C.c_void_p]
        for i in range(2):
            capi.lib().kvp_debug_proj_trace(buf[i].data_ptr())
            capi.call("kvp_matmul_packed", x.data_ptr(), B, K, pks[i % len(pks)].data_ptr(), N, out.data_ptr(), N, 0,
                      wsp.data_ptr(), None)
        torch.cuda.synchronize()
        capi.lib().kvp_debug_proj_trace(None)
        t = buf.view(2, 160, 8).double().cpu()
        t0 = t[0, :, 0][t[0, :, 0] > 0].min()
        names = ["start", "setup", "pre-issued", "dep-wait done", "first full", "last mma", "epi done", "end"]
        for i in range(2):
            v = t[i][t[i, :, 0] > 0]
            print(f"launch {i}: " + "  ".join(f"{n} {((v[:, k] - t0) / 1e3).median().item():.2f}/{((v[:, k] - t0) / 1e3).max().item():.2f}" for k, n in enumerate(names)))
    ref = x.float() @ ws_[-1].float()
    res["rel_err"] = ((out - ref).abs().max() / ref.abs().max()).item()
    print(json.dumps(dict(B=B, K=K, N=N, **res)))


if __name__ == "__main__":
    main()
