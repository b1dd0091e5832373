"""GPU parity at every BASELINE configuration against the compiled reference
(oracle/_ref: the reference's own C++ sources), not a restatement.

* C1 (BASELINE configs[0]): LLaVA-1.5-7B single layer, 32 heads x 128 dim,
  576 visual + 64 text tokens, rank 16, fp32 — the reference's own cache
  (latent-factor workload, compress_now) replayed through kvp_attend_plan;
  bar SURVEY §7.2: context <= 1e-4 * max(1, |oracle|), head_avg rows sum to
  1 +- 1e-6.
* C2/C3/C4 (2x/4x/8x)/C5 shapes: the fused tcgen05 serving kernel
  (kvp_decode_fused) against the reference's attend_materialized on the same
  bf16-rounded factors installed into a reference LayerCache (bar 1e-3), plus
  the reference's update_importance on its head average (EMA, 1e-6).
* Philox: device gaussian_matrix vs the reference generator (tests/golden/rng.npz).
* Compaction at the C2 shape: reconstruction error <= 1.02x the reference's
  own randomized SVD on the same matrix, right rows orthonormal.
"""
from __future__ import annotations

import ctypes as C
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from kvp_testlib import bf16_round, run_fused

pytestmark = pytest.mark.gpu


def _torch():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _ref():
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    return ref


# ---------------------------------------------------------------------------
# C1: the reference's own cache through the generic plan kernel (fp32)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("seed", [11, 21, 31])
def test_c1_attend_plan_matches_reference(seed):
    _torch()
    ref = _ref()
    from oracle import cases
    from oracle import kvpack_oracle as ko
    from kvp_testlib import attend_on_gpu
    H, Hkv, D, n_vis, n_txt, R = 32, 32, 128, 576, 64, 16
    cache = ref.RefCache(H, Hkv, D, dtype="f32")
    # latent-factor workload (harness.cpp:82-128): visual {2R, 0.98, R, 1e-2}, textual default {48, 0.98, 4, 1e-2}
    for mod, (T, tr, sh) in ((0, (n_vis, 2 * R, R)), (1, (n_txt, 48, 4))):
        k = ref.latent_factor_matrix(T, H, Hkv, D, tr, 0.98, sh, 1e-2, seed, ko.stream_id(2, 0, 0, 2 * mod))
        v = ref.latent_factor_matrix(T, H, Hkv, D, tr, 0.98, sh, 1e-2, seed, ko.stream_id(2, 0, 0, 2 * mod + 1))
        cache.append(mod, k, v)
    ini = cases.decode_ini(ranks=(R, R, 0, 0), svd="exact")
    cache.compress_now(ini)
    rng = np.random.default_rng(seed)
    pos, _ = cache.importance()
    cache.set_importance(rng.uniform(0, 1, pos.size))
    st = cases.export_state(cache)
    _, _, nxt = cache.segment_info(0)
    q = rng.standard_normal((1, H * D)).astype(np.float32).astype(np.float64)
    qpos = np.array([nxt], dtype=np.uint64)
    rctx, rha, plan = cache.attend(q, qpos, ini)
    ctx, ha, hat = attend_on_gpu(st, plan, q, qpos, dtype="f32")
    err = np.abs(ctx - rctx).max() / max(1.0, np.abs(rctx).max())
    print(f"C1 seed {seed}: plan {len(plan)} entries, context rel err {err:.2e}, "
          f"head_avg err {np.abs(ha - rha).max():.2e}")
    assert err <= 1e-4
    assert np.abs(ha.sum(axis=1) - 1.0).max() <= 1e-6
    assert np.abs(ha - rha).max() <= 1e-6
    # table-order head average (the EMA's input, decoder.cpp:592-601) is the plan-order one un-permuted
    tpos = {int(p): i for i, p in enumerate(st["imp_positions"])}
    back = np.zeros_like(hat)
    for j, e in enumerate(plan):
        back[:, tpos[int(e[5])]] = ha[:, j]
    assert np.array_equal(back, hat)


# ---------------------------------------------------------------------------
# Fused serving kernel at the BASELINE shapes vs the reference's attend
# ---------------------------------------------------------------------------
CONFIG_SHAPES = {
    # name: B, H, Hkv, D, n_comp, rank, n_tail, cap (one instance: the reference attend is ~10 s per instance)
    "c2": (1, 32, 32, 128, 2304, 368, 65, 320),
    "c3": (1, 40, 40, 128, 4096, 284, 320, 320),
    "c4_8x": (1, 32, 32, 128, 4096, 256, 80, 320),
    "c4_4x": (1, 32, 32, 128, 4096, 512, 80, 320),
    "c4_2x": (1, 32, 32, 128, 4096, 1024, 80, 320),
    "c5": (1, 32, 32, 128, 2048, 128, 200, 320),
}


def _reference_attend(ref, case, b, H, Hkv, D, nt):
    """The reference attend_materialized + update_importance on the case's
    bf16-rounded factors and tail (identical inputs)."""
    from oracle import cases
    W = Hkv * D
    n, rk = case["left_k"].shape[1:]
    rv = case["left_v"].shape[2]
    cache = ref.RefCache(H, Hkv, D, dtype="f64")
    cache.append(0, np.zeros((n, W)), np.zeros((n, W)))  # positions 0..n-1; rows replaced by the factors
    cache.factor_tail(0, (case["left_k"][b], case["right_k"][b]), (case["left_v"][b], case["right_v"][b]))
    cache.append(1, case["tail_k"][b, :nt], case["tail_v"][b, :nt])
    cache.set_importance(case["imp"][b, :n + nt])
    ini = cases.decode_ini(ranks=(rk, rv, 0, 0))
    qpos = np.array([n + nt], dtype=np.uint64)
    ctx, ha, plan = cache.attend(case["q"][b:b + 1], qpos, ini)
    ema = ref.update_importance(case["imp"][b, :n + nt], ha, 0.25)  # plan order == table order here
    return ctx[0], ha[0], ema, plan


@pytest.mark.parametrize("name", sorted(CONFIG_SHAPES))
def test_fused_matches_reference_at_config_shape(name):
    _torch()
    ref = _ref()
    from kvp_testlib import make_case
    B, H, Hkv, D, n, r, nt, cap = CONFIG_SHAPES[name]
    rng = np.random.default_rng(abs(hash(name)) % 2**32)
    case = make_case(rng, B, H, Hkv, D, n, r, r, nt, cap)
    ctx, ha, imp = run_fused(case, H, Hkv, D, nt, 0.25, cluster=0)
    with ThreadPoolExecutor(max_workers=B) as pool:
        outs = list(pool.map(lambda b: _reference_attend(ref, case, b, H, Hkv, D, nt), range(B)))
    for b, (rctx, rha, rema, plan) in enumerate(outs):
        assert [int(e[5]) for e in plan] == list(range(n + nt))  # untiered plan: storage order
        err = np.abs(ctx[b] - rctx).max() / np.abs(rctx).max()
        print(f"{name}: context rel err {err:.2e}, head_avg err {np.abs(ha[b, :n + nt] - rha).max():.2e}, "
              f"EMA err {np.abs(imp[b, :n + nt] - rema).max():.2e}")
        assert err <= 1e-3
        assert np.abs(ha[b, :n + nt] - rha).max() <= 1e-5
        assert np.abs(imp[b, :n + nt] - rema).max() <= 1e-5
        assert np.array_equal(imp[b, n + nt:], case["imp"][b, n + nt:])


# ---------------------------------------------------------------------------
# Philox Gaussian generator, bit-level, against the reference's own draws
# ---------------------------------------------------------------------------
def test_device_philox_matches_reference(golden):
    torch = _torch()
    from paper_2603_23914_b200 import _capi as capi
    g = golden("rng")
    for i, (seed, stream) in enumerate(g["streams"]):
        want = g[f"gauss_{i}"]
        out64 = torch.empty(want.size, dtype=torch.float64, device="cuda")
        out32 = torch.empty(want.size, dtype=torch.float32, device="cuda")
        for dt, out in ((capi.KVP_F64, out64), (capi.KVP_F32, out32)):
            capi.call("kvp_gaussian_matrix", C.c_int64(1), C.c_int64(want.size), C.c_uint64(int(seed)),
                      C.c_uint64(int(stream)), dt, out.data_ptr(), None)
        torch.cuda.synchronize()
        got64, got32 = out64.cpu().numpy(), out32.cpu().numpy()
        # f64: identical Philox words and Box-Muller; only the device libm's log/cos/sin may differ by an ulp
        ulps = np.abs(got64.view(np.int64) - want.view(np.int64))
        exact = int((ulps == 0).sum())
        print(f"stream {i}: f64 exact {exact}/{want.size}, max ulp {int(ulps.max())}")
        assert ulps.max() <= 4
        # f32 (the reference's float instantiation casts the same double): bit-exact
        assert np.array_equal(got32, want.astype(np.float32))


# ---------------------------------------------------------------------------
# Compaction accuracy at the C2 shape vs the reference's randomized SVD
# ---------------------------------------------------------------------------
def test_compaction_c2_shape_within_1p02_of_reference():
    torch = _torch()
    ref = _ref()
    from paper_2603_23914_b200 import kvpack
    from oracle import kvpack_oracle as ko
    T, H, D, R = 2304, 32, 128, 368
    W = H * D
    a = ref.latent_factor_matrix(T, H, H, D, 2 * R, 0.98, R, 1e-2, 11, ko.stream_id(2, 0, 0, 0))
    left, right = kvpack.truncated_svd(a, R, method="randomized", seed=0)
    err = np.linalg.norm(a - left @ right) / np.linalg.norm(a)
    rl, rr = ref.truncated_svd(a, R, method="randomized", seed=0)
    ref_err = np.linalg.norm(a - rl @ rr) / np.linalg.norm(a)
    orth = np.abs(right @ right.T - np.eye(R)).max()
    print(f"C2 compaction: rel err {err:.5f} vs reference {ref_err:.5f} (ratio {err / ref_err:.4f}), "
          f"|right right^T - I| {orth:.2e}")
    assert err <= 1.02 * ref_err
    assert orth <= 1e-4


def test_compaction_c4_4x_shape_within_1p02_of_reference():
    # C4 4x (Qwen-VL-shaped 4096 x 4096 segment, rank 512): the sketch (520) spans two 384-column
    # tensor-core blocks and the 520 x 520 eigenproblem 36 Jacobi blocks
    _torch()
    ref = _ref()
    from paper_2603_23914_b200 import kvpack
    from oracle import kvpack_oracle as ko
    T, H, D, R = 4096, 32, 128, 512
    a = ref.latent_factor_matrix(T, H, H, D, 2 * R, 0.98, R, 1e-2, 11, ko.stream_id(2, 0, 0, 0))
    left, right = kvpack.truncated_svd(a, R, method="randomized", seed=0)
    err = np.linalg.norm(a - left @ right) / np.linalg.norm(a)
    rl, rr = ref.truncated_svd(a, R, method="randomized", seed=0)
    ref_err = np.linalg.norm(a - rl @ rr) / np.linalg.norm(a)
    orth = np.abs(right @ right.T - np.eye(R)).max()
    print(f"C4 4x compaction: rel err {err:.5f} vs reference {ref_err:.5f} (ratio {err / ref_err:.4f}), "
          f"|right right^T - I| {orth:.2e}")
    assert err <= 1.02 * ref_err
    assert orth <= 1e-4
