"""ORACLE / TEST INFRASTRUCTURE ONLY.

Seeded scenario builders shared by the golden-fixture generator and the GPU
parity tests.  A scenario drives the *reference* (``oracle.ref.RefCache``)
through its own API — append_tokens, compress_now, importance scores — and
exports the resulting cache state (factors, tails, positions, scores) plus
the reference outputs, so the CUDA path can be fed the identical state.
"""
from __future__ import annotations

import numpy as np

from . import ref


def decode_ini(ranks=(8, 8, 0, 0), tiering=None, period=None, svd="exact", fused=False, tile=64,
               alpha=0.25, extra=""):
    lines = ["[decode]"]
    lines.append(f"compression_period = {'none' if period is None else period}")
    lines.append(f"svd_method = {svd}")
    lines.append(f"alpha = {alpha!r}")
    lines.append(f"fused = {'true' if fused else 'false'}")
    lines.append(f"fused_tile = {tile}")
    lines += extra.splitlines()
    lines += ["[decode.ranks]", f"key_visual = {ranks[0]}", f"value_visual = {ranks[1]}",
              f"key_textual = {ranks[2]}", f"value_textual = {ranks[3]}"]
    if tiering is not None:
        r, kf, vf = tiering
        lines += ["[decode.tiering]", "ratios = " + ", ".join(repr(x) for x in r),
                  "key_rank_fractions = " + ", ".join(repr(x) for x in kf),
                  "value_rank_fractions = " + ", ".join(repr(x) for x in vf)]
    return "\n".join(lines) + "\n"


def planted(rows, cols, rank, rng, decay=0.7):
    m = np.zeros((rows, cols))
    w = 1.0
    for _ in range(rank):
        m += w * np.outer(rng.standard_normal(rows), rng.standard_normal(cols))
        w *= decay
    return m


def export_state(cache: ref.RefCache):
    """Flatten a reference LayerCache into arrays (segment 0 visual, 1 textual)."""
    st = {"H": cache.H, "Hkv": cache.Hkv, "D": cache.D}
    pos, sc = cache.importance()
    st["imp_positions"], st["imp_scores"] = pos, sc
    for s in (0, 1):
        nb, tl, _ = cache.segment_info(s)
        st[f"s{s}_nblocks"] = nb
        for b in range(nb):
            for kind, kn in ((0, "k"), (1, "v")):
                form, a, bmat, p = cache.block(s, b, kind)
                if form == "lowrank":
                    st[f"s{s}b{b}_{kn}_left"], st[f"s{s}b{b}_{kn}_right"] = a, bmat
                else:
                    st[f"s{s}b{b}_{kn}_rows"] = a
                st[f"s{s}b{b}_positions"] = p
        k, v, p = cache.tail(s)
        st[f"s{s}_tail_k"], st[f"s{s}_tail_v"], st[f"s{s}_tail_positions"] = k, v, p
    return st


def attend_case(seed, geom=(4, 4, 8), n_vis=40, n_txt=6, rank=8, tq=2, tiering=None, dtype="f64",
                scale_q=1.0, planted_rank=True, ranks=None, random_scores=True):
    """Reference attend_{materialized,fused} on a mixed cache: a factored
    visual block (+ optional dense textual tail), like test_decoder.cpp:74-97."""
    H, Hkv, D = geom
    W = Hkv * D
    rng = np.random.default_rng(seed)
    cache = ref.RefCache(H, Hkv, D, dtype=dtype)
    if planted_rank:
        kv = planted(n_vis, W, rank, rng), planted(n_vis, W, rank, rng)
    else:
        kv = rng.standard_normal((n_vis, W)), rng.standard_normal((n_vis, W))
    cache.append(0, *kv)
    if n_txt:
        cache.append(1, rng.standard_normal((n_txt, W)), rng.standard_normal((n_txt, W)))
    ranks = ranks if ranks is not None else (rank, rank, 0, 0)
    ini = decode_ini(ranks=ranks, tiering=tiering)
    cache.compress_now(ini)
    if random_scores:
        pos, _ = cache.importance()
        sc = rng.uniform(0.0, 1.0, size=pos.size)
        sc[rng.integers(0, pos.size, size=max(1, pos.size // 8))] = 0.5  # force ties
        cache.set_importance(sc)
    st = export_state(cache)
    _, _, nxt = cache.segment_info(0)
    q = rng.standard_normal((tq, H * D)) * scale_q
    qpos = np.arange(nxt, nxt + tq, dtype=np.uint64)
    ctx, ha, plan = cache.attend(q, qpos, ini, fused=False)
    ctx_f, ha_f, _ = cache.attend(q, qpos, ini, fused=True, tile=7)
    st.update(queries=q, qpos=qpos, context=ctx, head_avg=ha, plan=plan, context_fused=ctx_f,
              head_avg_fused=ha_f, ini=np.array(ini), dtype=np.array(dtype))
    return st


def decode_case(seed, geom=(4, 4, 8), n_vis=48, n_txt=8, rank=8, steps=5, tiering=None, dtype="f64",
                period=None, ranks=None, svd="exact"):
    """Reference decode_step sequence after a prefill compress_now
    (harness.cpp:256-330 minus the dense chain)."""
    H, Hkv, D = geom
    W, HD = Hkv * D, H * D
    rng = np.random.default_rng(seed)
    cache = ref.RefCache(H, Hkv, D, dtype=dtype)
    cache.append(0, planted(n_vis, W, rank, rng), planted(n_vis, W, rank, rng))
    cache.append(1, rng.standard_normal((n_txt, W)), rng.standard_normal((n_txt, W)))
    ranks = ranks if ranks is not None else (rank, rank, 0, 0)
    ini = decode_ini(ranks=ranks, tiering=tiering, period=period, svd=svd)
    cache.compress_now(ini)
    st0 = export_state(cache)
    s = 1.0 / np.sqrt(HD)
    wq, wk, wv, wo = (rng.standard_normal(sh) * s for sh in ((HD, HD), (HD, W), (HD, W), (HD, HD)))
    xs = rng.standard_normal((steps, HD))
    outs, reps = [], []
    for t in range(steps):
        y, rep = cache.decode_step(xs[t:t + 1], wq, wk, wv, wo, ini)
        outs.append(y[0])
        reps.append([rep.bytes_before, rep.bytes_after, rep.importance_bytes, rep.decompress_flops,
                     rep.decompress_flops_full, rep.compression_event])
    pos, sc = cache.importance()
    st = {"state0_" + k: v for k, v in st0.items()}
    st.update(wq=wq, wk=wk, wv=wv, wo=wo, inputs=xs, outputs=np.array(outs), reports=np.array(reps, np.uint64),
              final_positions=pos, final_scores=sc, ini=np.array(ini), dtype=np.array(dtype))
    return st
