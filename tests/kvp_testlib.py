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
