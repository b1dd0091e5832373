"""Test helpers: feed a reference cache state (exported by oracle/cases.py or
stored in tests/golden) to the product C-ABI through torch device buffers."""
from __future__ import annotations

import ctypes as C

import numpy as np

from paper_2603_23914_b200 import _capi as capi

TORCH_DT = {"f64": "float64", "f32": "float32", "bf16": "bfloat16"}
KVP_DT = {"f64": capi.KVP_F64, "f32": capi.KVP_F32, "bf16": capi.KVP_BF16}


def dev(a, dtype="f64"):
    import torch
    return torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=getattr(torch, TORCH_DT[dtype]))


def stores_from_state(st, dtype):
    """Returns (stores list, keepalive tensors, index map {(seg, block|-1, kind): store})."""
    stores, keep, index = [], [], {}
    for s in (0, 1):
        for b in range(int(st[f"s{s}_nblocks"])):
            for kind, kn in ((0, "k"), (1, "v")):
                if f"s{s}b{b}_{kn}_left" in st:
                    left, right = dev(st[f"s{s}b{b}_{kn}_left"], dtype), dev(st[f"s{s}b{b}_{kn}_right"], dtype)
                    keep += [left, right]
                    stores.append(capi.Store(capi.KVP_LOWRANK, left.shape[1], left.data_ptr(), right.data_ptr(),
                                             left.shape[1], right.shape[1]))
                else:
                    rows = dev(st[f"s{s}b{b}_{kn}_rows"], dtype)
                    keep.append(rows)
                    stores.append(capi.Store(capi.KVP_DENSE, 0, rows.data_ptr(), None, rows.shape[1], 0))
                index[(s, b, kind)] = len(stores) - 1
        tk = st[f"s{s}_tail_k"]
        if tk.shape[0]:
            for kind, key in ((0, "tail_k"), (1, "tail_v")):
                rows = dev(st[f"s{s}_{key}"], dtype)
                keep.append(rows)
                stores.append(capi.Store(capi.KVP_DENSE, 0, rows.data_ptr(), None, rows.shape[1], 0))
                index[(s, -1, kind)] = len(stores) - 1
    return stores, keep, index


def attend_on_gpu(st, plan, queries, qpos, dtype="f64", with_table=True):
    import torch
    stores, keep, index = stores_from_state(st, dtype)
    tpos = {int(p): i for i, p in enumerate(st["imp_positions"])}
    ents = (capi.PlanEntry * len(plan))()
    for j, (seg, blk, row, rk, rv, pos) in enumerate(plan):
        e = ents[j]
        e.k_store, e.v_store = index[(int(seg), int(blk), 0)], index[(int(seg), int(blk), 1)]
        e.row, e.rank_k, e.rank_v = int(row), int(rk), int(rv)
        e.table_index = tpos.get(int(pos), -1)
        e.position = int(pos)
    H, Hkv, D = int(st["H"]), int(st["Hkv"]), int(st["D"])
    q = dev(queries, "f64")
    qp = torch.as_tensor(np.asarray(qpos, dtype=np.int64)).cuda()
    tq, n = q.shape[0], len(plan)
    ctx = torch.zeros((tq, H * D), dtype=torch.float64, device="cuda")
    ha = torch.zeros((tq, n), dtype=torch.float64, device="cuda")
    tsize = len(tpos) if with_table else 0
    hat = torch.zeros((tq, max(tsize, 1)), dtype=torch.float64, device="cuda")
    sarr = (capi.Store * len(stores))(*stores)
    d = capi.AttendDesc(H, Hkv, D, KVP_DT[dtype], len(stores), n, tq, tsize, sarr, ents, q.data_ptr(),
                        qp.data_ptr(), ctx.data_ptr(), ha.data_ptr(), hat.data_ptr() if with_table else None)
    capi.call("kvp_attend_plan", C.byref(d), None)
    torch.cuda.synchronize()
    del keep
    return ctx.cpu().numpy(), ha.cpu().numpy(), hat.cpu().numpy()[:, :tsize]


# ---------------------------------------------------------------------------
# Fused serving kernel (kvp_decode_fused) helpers: a synthetic bf16 serving
# cache, the fp64 dense oracle over the same rounded factors, and one call.
# ---------------------------------------------------------------------------
from paper_2603_23914_b200._capi import FusedDesc  # noqa: E402


def bf16_round(x):
    import torch
    return torch.as_tensor(x, dtype=torch.float32).to(torch.bfloat16).to(torch.float64).numpy()


def make_case(rng, B, H, Hkv, D, n, rk, rv, nt, cap):
    W = Hkv * D
    def orth(r):
        q, _ = np.linalg.qr(rng.standard_normal((W, r)))
        return q.T
    case = dict(
        left_k=bf16_round(rng.standard_normal((B, n, rk)) * np.linspace(3, 0.3, rk)),
        left_v=bf16_round(rng.standard_normal((B, n, rv)) * np.linspace(3, 0.3, rv)),
        right_k=bf16_round(np.stack([orth(rk) for _ in range(B)])),
        right_v=bf16_round(np.stack([orth(rv) for _ in range(B)])),
        tail_k=bf16_round(rng.standard_normal((B, cap, W))),
        tail_v=bf16_round(rng.standard_normal((B, cap, W))),
        q=rng.standard_normal((B, H * D)).astype(np.float32).astype(np.float64) * 2.0,
        imp=rng.uniform(0, 1, (B, n + cap)),
    )
    return case


def oracle(case, H, Hkv, D, nt, alpha, tier=None, rv2=0):
    B, n, _ = case["left_k"].shape
    per = H // Hkv
    ctx = np.zeros((B, H * D))
    ha = np.zeros((B, n + nt))
    imp = case["imp"].copy()
    for b in range(B):
        K = np.concatenate([case["left_k"][b] @ case["right_k"][b], case["tail_k"][b, :nt]])
        Vc = case["left_v"][b] @ case["right_v"][b]
        if tier is not None:  # second-tier tokens: value-rank prefix rv2 (store_decompress_row, cache.cpp:63-101)
            t2 = tier[b] != 0
            Vc[t2] = case["left_v"][b][t2, :rv2] @ case["right_v"][b][:rv2]
        V = np.concatenate([Vc, case["tail_v"][b, :nt]])
        for h in range(H):
            g = h // per
            s = K[:, g * D:(g + 1) * D] @ case["q"][b, h * D:(h + 1) * D] / np.sqrt(D)
            e = np.exp(s - s.max())
            z = e.sum()
            ctx[b, h * D:(h + 1) * D] = e @ V[:, g * D:(g + 1) * D] / z
            ha[b] += e / z / H
        cols = np.r_[np.arange(n), n + np.arange(nt)]
        imp[b, cols] = alpha * imp[b, cols] + (1 - alpha) * ha[b]
    return ctx, ha, imp


def run_fused(case, H, Hkv, D, nt, alpha, cluster=0, ld_pad=8, tier=None, rv2=0):
    import torch
    from paper_2603_23914_b200 import _capi as capi
    B, n, rk = case["left_k"].shape
    rv = case["left_v"].shape[2]
    cap = case["tail_k"].shape[1]
    def left(x):  # row-major bf16 -> packed panel-major layout (kvp_pack_left)
        src = torch.as_tensor(x).to(torch.bfloat16).cuda().contiguous()
        r = x.shape[2]
        out = torch.zeros(capi.lib().kvp_packed_left_bytes(B, n, r), dtype=torch.uint8, device="cuda")
        capi.call("kvp_pack_left", src.data_ptr(), r, B, n, r, out.data_ptr(), None)
        return out
    bf = lambda x: torch.as_tensor(x).to(torch.bfloat16).cuda().contiguous()
    t = dict(lk=left(case["left_k"]), lv=left(case["left_v"]), rk=bf(case["right_k"]), rv=bf(case["right_v"]),
             tk=bf(case["tail_k"]), tv=bf(case["tail_v"]), q=torch.as_tensor(case["q"], dtype=torch.float32).cuda(),
             imp=torch.as_tensor(case["imp"]).cuda().contiguous())
    ctx = torch.zeros((B, H * D), dtype=torch.float32, device="cuda")
    ha = torch.zeros((B, n + cap), dtype=torch.float32, device="cuda")
    d = FusedDesc(H, Hkv, D, B, n, rk, rv, 0, cap, nt, None, cluster, 0, t["lk"].data_ptr(), t["rk"].data_ptr(),
                  t["lv"].data_ptr(), t["rv"].data_ptr(), t["tk"].data_ptr(), t["tv"].data_ptr(), t["q"].data_ptr(),
                  t["imp"].data_ptr(), n + cap, alpha, ha.data_ptr(), ctx.data_ptr())
    if tier is not None:
        t["tier"] = torch.as_tensor(np.ascontiguousarray(tier, dtype=np.uint8)).cuda()
        d.tier2_value_rank = rv2
        d.value_tier = t["tier"].data_ptr()
    capi.lib().kvp_decode_fused.argtypes = [C.POINTER(FusedDesc), C.c_void_p]
    capi.check(capi.lib().kvp_decode_fused(C.byref(d), None))
    torch.cuda.synchronize()
    return ctx.cpu().numpy().astype(np.float64), ha.cpu().numpy().astype(np.float64), t["imp"].cpu().numpy()


