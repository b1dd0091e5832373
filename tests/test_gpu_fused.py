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


from kvp_testlib import bf16_round, make_case, oracle, run_fused  # noqa: E402,F401


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
