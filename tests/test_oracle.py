"""CPU tests: the numpy restatement (oracle/kvpack_oracle.py) pinned against
the reference's own known-answer tests and the golden vectors the compiled
reference produced (tests/golden, oracle/gen_golden.py)."""
import glob

import numpy as np
import pytest

from oracle import kvpack_oracle as ko
from pathlib import Path

GOLDEN = Path(__file__).resolve().parent / "golden"


# --- known answers from the reference's unit tests --------------------------

def test_philox_known_answer_blocks():
    # test_rng.cpp:14-30
    cases = [((0, 0), (0, 0, 0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
             ((0xFFFFFFFF, 0xFFFFFFFF), (0xFFFFFFFF,) * 4, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
             ((0xA4093822, 0x299F31D0), (0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344),
              (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
             ((123, 456), (1, 0, 0, 7), (0x4F61938B, 0x9357F452, 0xED08E3E3, 0x494E8DA4))]
    for key, ctr, want in cases:
        got = ko.philox_round10(key, [np.array([c], dtype=np.uint64) for c in ctr])
        assert tuple(int(x[0]) for x in got) == want


def test_closed_forms():
    # test_cache.cpp:191-196, test_importance.cpp:138-157
    assert ko.compression_ratio(1000, 5120, 64) == 13.071895424836601
    assert ko.compression_ratio(576, 4096, 64) == 7.890410958904109
    assert ko.compression_ratio(64, 128, 16) == 2.6666666666666665
    assert ko.compression_ratio(100, 64, 0) == 1.0
    flops, red = ko.flops_partial_decompress(1000, 5120, [0.1, 0.9], [64, 16])
    assert flops == 212992000 and abs(red - 0.675) <= 1e-15
    assert ko.flops_partial_decompress(50, 32, [1.0], [16]) == (2 * 50 * 32 * 16, 0.0)


def test_ema_hand_cases():
    # test_importance.cpp:31-50
    assert ko.update_importance([0.8, 0.2], [[0.0, 1.0]], 0.25)[0] == pytest.approx(0.2, abs=1e-15)
    out = ko.update_importance([0.4, 0.6], [[0.1, 0.9], [0.1, 0.9]], 0.25)
    assert out[0] == pytest.approx(0.11875, abs=1e-15)
    assert list(ko.update_importance([0.9, 0.1], [[0.3, 0.7]], 0.0)) == [0.3, 0.7]
    assert list(ko.update_importance([0.9, 0.1], [[0.3, 0.7]], 1.0)) == [0.9, 0.1]
    with pytest.raises(ValueError):
        ko.update_importance([0.5, 0.5], [[0.9, 0.3]], 0.25)


def test_group_known_answers():
    # test_importance.cpp:85-130
    t = ko.assign_groups([0.9, 0.01, 0.02, 0.03, 0.02, 0.01, 0.02, 0.8], [0.25, 0.75], [16, 8])
    assert list(ko.masks_from_tiers(t, 2)[0]) == [0, 7]
    t = ko.assign_groups([0.4] * 4, [0.5, 0.5], [16, 8])
    assert [list(m) for m in ko.masks_from_tiers(t, 2)] == [[0, 1], [2, 3]]
    t = ko.assign_groups(0.01 * np.arange(10), [0.3, 0.3, 0.4], [32, 16, 8])
    assert [len(m) for m in ko.masks_from_tiers(t, 3)] == [3, 3, 4]
    with pytest.raises(ValueError):
        ko.assign_groups([0.1, 0.2], [0.5, 0.4], [16, 8])


def test_tier_rank_resolution():
    # test_decoder.cpp:246-265
    assert [ko.resolved_tier_rank(f, 16) for f in (1.0, 0.5, 0.125)] == [16, 8, 2]
    assert [ko.resolved_tier_rank(f, 16) for f in (1.0, 0.25, 0.125)] == [16, 4, 2]
    assert ko.group_sizes(32, [0.25, 0.5, 0.25]) == [8, 16, 8]


# --- golden vectors from the compiled reference -----------------------------

def test_gaussian_stream_matches_reference(golden):
    g = golden("rng")
    for i, (seed, stream) in enumerate(g["streams"]):
        np.testing.assert_allclose(ko.philox_gaussians(int(seed), int(stream), 257), g[f"gauss_{i}"],
                                   rtol=0, atol=1e-14)


def test_latent_factor_matrix_matches_reference(golden):
    g = golden("rng")
    tok, _, kvh, d, r, sh, seed, stream = (int(x) for x in g["lfm_args"])
    out = ko.latent_factor_matrix(tok, kvh, d, r, 0.9, sh, 0.01, seed, stream)
    np.testing.assert_allclose(out, g["lfm"], rtol=0, atol=1e-12)


def test_assign_groups_bit_exact_vs_reference(golden):
    g = golden("importance")
    for k in range(int(g["n_groups"])):
        tier = ko.assign_groups(g[f"g{k}_scores"], list(g[f"g{k}_ratios"]), [int(x) for x in g[f"g{k}_ranks"]])
        assert np.array_equal(tier, g[f"g{k}_tier"]), k


def test_ema_bit_exact_vs_reference(golden):
    g = golden("importance")
    for k in range(int(g["n_ema"])):
        out = ko.update_importance(g[f"e{k}_scores"], g[f"e{k}_attn"], float(g[f"e{k}_alpha"]))
        assert np.array_equal(out, g[f"e{k}_out"]), k


def _segments(st):
    segs = []
    for s in (0, 1):
        seg = ko.Segment()
        for b in range(int(st[f"s{s}_nblocks"])):
            stores = []
            for kn in ("k", "v"):
                if f"s{s}b{b}_{kn}_left" in st:
                    stores.append(ko.Store(left=st[f"s{s}b{b}_{kn}_left"], right=st[f"s{s}b{b}_{kn}_right"]))
                else:
                    stores.append(ko.Store(rows=st[f"s{s}b{b}_{kn}_rows"]))
            seg.blocks.append(ko.Block(st[f"s{s}b{b}_positions"], *stores))
        seg.tail_k, seg.tail_v = st[f"s{s}_tail_k"], st[f"s{s}_tail_v"]
        seg.tail_positions = st[f"s{s}_tail_positions"]
        segs.append(seg)
    return segs


def _tiering(ini):
    lines = dict(l.split(" = ") for l in str(ini).splitlines() if " = " in l)
    if "ratios" not in lines:
        return None
    f = lambda k: [float(x) for x in lines[k].split(",")]
    return ko.Tiering(f("ratios"), f("key_rank_fractions"), f("value_rank_fractions"))


@pytest.mark.parametrize("path", sorted(glob.glob(str(GOLDEN / "attend_*.npz"))))
def test_attend_restatement_vs_reference(path):
    st = dict(np.load(path))
    segs = _segments(st)
    scores = dict(zip((int(p) for p in st["imp_positions"]), st["imp_scores"]))
    plan = ko.build_retrieval_plan(segs, scores, _tiering(st["ini"]))
    assert np.array_equal(plan, st["plan"])  # retrieval plan: bit-exact
    ctx, ha = ko.attend_lowrank(segs, plan, st["queries"], st["qpos"], int(st["H"]), int(st["Hkv"]), int(st["D"]))
    tol = 1e-4 if str(st["dtype"]) == "f32" else 1e-10
    scale = max(1.0, np.abs(st["context"]).max())
    assert np.abs(ctx - st["context"]).max() <= tol * scale
    assert np.abs(ha - st["head_avg"]).max() <= tol
    # fused (tile 7) vs materialized inside the reference itself
    assert np.abs(st["context_fused"] - st["context"]).max() <= 1e-6 * scale


def test_svd_restatement_vs_reference(golden):
    g = golden("svd")
    for name in g["names"]:
        a, r = g[f"{name}_a"], int(g[f"{name}_rank"])
        np.testing.assert_allclose(np.linalg.svd(a, compute_uv=False), g[f"{name}_sv"], rtol=1e-12, atol=1e-12)
        for method in ("exact", "randomized"):
            left, right = ko.truncated_svd(a, r, method=method, seed=7)
            err = np.linalg.norm(a - left @ right)
            assert err == pytest.approx(float(g[f"{name}_{method}_err"]), rel=1e-6, abs=1e-9)
            assert np.allclose(right @ right.T, np.eye(r), atol=1e-10)
