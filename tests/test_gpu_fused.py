"""GPU parity of the fused cluster/tcgen05 decode kernel (kvp_decode_fused).

Oracle: fp64 dense attention over K~ = [left_k right_k ; tail_k] and
V~ = [left_v right_v ; tail_v] built from the *same bf16-rounded* factors
(SURVEY.md §8c parity protocol: identical rounded inputs, bf16 bound 1e-3),
plus the reference EMA (importance.cpp:33-65) on the head-averaged rows."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _torch():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


from paper_2603_23914_b200._capi import FusedDesc  # noqa: E402


def bf16_round(x):
    torch = _torch()
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
    torch = _torch()
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


SHAPES = [
    # B, H, Hkv, D, n_comp, rank_k, rank_v, n_tail, cap, cluster
    (2, 32, 32, 128, 2304, 368, 368, 65, 320, 8),   # C2 geometry (4x compression), first decode step
    (2, 40, 40, 128, 4096, 284, 284, 320, 320, 8),  # C3 geometry (8x), last decode step
    (1, 32, 32, 128, 2048, 128, 128, 200, 320, 8),  # C5 geometry
    (2, 32, 32, 128, 2304, 368, 368, 66, 320, 0),   # C2, occupancy-chosen cluster (the engine's choice)
    (1, 32, 32, 128, 4096, 256, 256, 80, 320, 0),   # C4 8x
    (1, 32, 32, 128, 4096, 512, 512, 80, 320, 0),   # C4 4x
    (1, 32, 32, 128, 4096, 768, 768, 80, 320, 8),   # stacked hi/lo tiles exceed TMEM: two-MMA fallback
    (1, 32, 32, 128, 4096, 1024, 1024, 80, 320, 0), # C4 2x: p tiles over the dead P image (shared memory)
    (3, 8, 4, 64, 300, 40, 24, 5, 16, 8),           # GQA, ragged: idle CTAs, partial tiles, odd ranks
    (2, 16, 16, 128, 1000, 100, 70, 0, 8, 4),       # no tail, cluster of 4
]


@pytest.mark.parametrize("shape", SHAPES)
def test_fused_matches_fp64_oracle(shape):
    B, H, Hkv, D, n, rk, rv, nt, cap, cl = shape
    rng = np.random.default_rng(hash(shape) % 2**32)
    case = make_case(rng, B, H, Hkv, D, n, rk, rv, nt, cap)
    alpha = 0.25
    ctx, ha, imp = run_fused(case, H, Hkv, D, nt, alpha, cluster=cl)
    rctx, rha, rimp = oracle(case, H, Hkv, D, nt, alpha)
    scale = np.abs(rctx).max()
    err = np.abs(ctx - rctx).max() / scale
    print(f"shape {shape}: context max rel err {err:.3e}, head_avg max abs err "
          f"{np.abs(ha[:, np.r_[np.arange(n), n + np.arange(nt)]] - rha).max():.3e}")
    assert err <= 1e-3, f"context rel err {err:.3e}"
    cols = np.r_[np.arange(n), n + np.arange(nt)]
    assert np.abs(ha[:, cols] - rha).max() <= 1e-4
    assert np.allclose(ha[:, cols].sum(axis=1), 1.0, atol=1e-4)
    assert np.abs(imp - rimp).max() <= 1e-4
    untouched = np.setdiff1d(np.arange(n + cap), cols)
    assert np.array_equal(imp[:, untouched], case["imp"][:, untouched])


TIERED = [
    # B, H, Hkv, D, n_comp, rank, n_tail, cap, cluster, r1, value fraction of tier 2
    (1, 32, 32, 128, 2048, 128, 200, 320, 0, 0.25, 0.25),   # C5: VideoLLaVA 8 frames, paper tiering
    (2, 32, 32, 128, 2048, 128, 70, 320, 8, 0.125, 0.25),
    (2, 32, 32, 128, 2304, 368, 66, 320, 0, 0.5, 0.25),     # tier boundary inside the first of three U row tiles
    (1, 32, 32, 128, 4096, 284, 80, 320, 0, 0.375, 0.5),    # second-tier rank 142 spans two U row tiles
]


@pytest.mark.parametrize("shape", TIERED)
def test_fused_two_tier_values_match_oracle(shape):
    # Attention-aware decompression (decoder.cpp:105-188): tokens outside the
    # first group (assign_groups by importance, importance.cpp:67-117) use the
    # value-rank prefix resolved_tier_rank(fraction, rank) (decoder.cpp:18-23);
    # key fractions are 1.
    from oracle import kvpack_oracle as ko
    B, H, Hkv, D, n, r, nt, cap, cl, r1, vf = shape
    rng = np.random.default_rng(hash(shape) % 2**32)
    case = make_case(rng, B, H, Hkv, D, n, r, r, nt, cap)
    rv2 = ko.resolved_tier_rank(vf, r)
    tier = np.stack([ko.assign_groups(case["imp"][b, :n], [r1, 1.0 - r1], [r, rv2]) for b in range(B)])
    ctx, ha, imp = run_fused(case, H, Hkv, D, nt, 0.25, cluster=cl, tier=tier, rv2=rv2)
    rctx, rha, rimp = oracle(case, H, Hkv, D, nt, 0.25, tier=tier, rv2=rv2)
    err = np.abs(ctx - rctx).max() / np.abs(rctx).max()
    print(f"tiered {shape}: rv2 {rv2}, tier-2 tokens {int((tier != 0).sum())}, context max rel err {err:.3e}")
    assert err <= 1e-3
    cols = np.r_[np.arange(n), n + np.arange(nt)]
    assert np.abs(ha[:, cols] - rha).max() <= 1e-4
    assert np.abs(imp - rimp).max() <= 1e-4
    # the tiered output differs from the untiered one (the test exercises the second tier)
    uctx, _, _ = oracle(case, H, Hkv, D, nt, 0.25)
    assert np.abs(uctx - rctx).max() / np.abs(rctx).max() > 1e-2
