"""GPU parity of the drop-in cache API (kvp_cache_* / kvp_decode_step /
kvp_compress_now) against the compiled reference.

* The reference's decode goldens (tests/golden/decode_*.npz, written by
  oracle/gen_golden.py from oracle/_ref): the reference's post-prefill
  LayerCache is uploaded, the device decode_step runs the same inputs, and the
  outputs, StepReport integer fields and final importance table are compared.
* The reference's own decode loop with the device step substituted, side by
  side with oracle/_ref decode_step, including periodic joint re-factorisation
  (tail >= period; decoder.cpp:604-610) with compression events, separate
  epochs, tiering and a 600-step run with period 512.
* compress_now / segment_full_matrix on the device vs the reference.
"""
from __future__ import annotations

import numpy as np
import pytest

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


def _state(g, prefix="state0_"):
    return {k[len(prefix):]: v for k, v in g.items() if k.startswith(prefix)}


@pytest.mark.parametrize("name,tol", [("decode_plain", 1e-9), ("decode_gqa_tiers", 1e-9), ("decode_f32", 2e-5)])
def test_decode_goldens(golden, name, tol):
    _torch()
    from paper_2603_23914_b200 import cache as kc
    g = golden(name)
    dtype = str(g["dtype"])
    cfg = kc.DecodeConfig.from_ini(str(g["ini"]))
    cache = kc.LayerCacheBatch.from_state([_state(g)], dtype=dtype)
    w = kc.AttentionWeights(g["wq"], g["wk"], g["wv"], g["wo"], dtype=dtype)
    for t in range(g["inputs"].shape[0]):
        out, reps = kc.decode_step(g["inputs"][t:t + 1], cache, w, cfg)
        y = out.cpu().numpy()[0, 0]
        want = g["outputs"][t]
        err = np.abs(y - want).max() / max(1.0, np.abs(want).max())
        r = reps[0]
        got = [r.bytes_before, r.bytes_after, r.importance_bytes, r.decompress_flops, r.decompress_flops_full,
               int(r.compression_event)]
        print(f"{name} step {t}: output rel err {err:.2e}, report {got}")
        assert err <= tol
        assert got == [int(x) for x in g["reports"][t]]  # StepReport integer fields: bit-exact
        assert r.step == t
    pos, sc = cache.importance()
    assert np.array_equal(pos, g["final_positions"])
    assert np.abs(sc[0] - g["final_scores"]).max() <= (1e-12 if dtype == "f64" else 1e-6)


def _side_by_side(geom, n_vis, n_txt, ranks, steps, period, dtype, tiering=None, recompress="joint", seed=3,
                  batch=2, rank=8, check_every=1):
    """Reference caches (one per instance) and one device batch with identical post-prefill state; then the
    reference decode loop and the device decode_step on the same inputs."""
    ref = _ref()
    torch = _torch()
    from oracle import cases
    from paper_2603_23914_b200 import cache as kc
    H, Hkv, D = geom
    W, HD = Hkv * D, H * D
    rng = np.random.default_rng(seed)
    ini = cases.decode_ini(ranks=ranks, tiering=tiering, period=period, extra=f"recompress = {recompress}")
    refs, states = [], []
    for b in range(batch):
        c = ref.RefCache(H, Hkv, D, dtype=dtype)
        c.append(0, cases.planted(n_vis, W, rank - 2, rng), cases.planted(n_vis, W, rank - 2, rng))
        c.append(1, rng.standard_normal((n_txt, W)), rng.standard_normal((n_txt, W)))
        c.compress_now(ini)
        refs.append(c)
        states.append(cases.export_state(c))
    cfg = kc.DecodeConfig.from_ini(ini)
    dev = kc.LayerCacheBatch.from_state(states, dtype=dtype)
    s = 1.0 / np.sqrt(HD)
    wq, wk, wv, wo = (rng.standard_normal(sh) * s for sh in ((HD, HD), (HD, W), (HD, W), (HD, HD)))
    w = kc.AttentionWeights(wq, wk, wv, wo, dtype=dtype)
    xs = rng.standard_normal((steps, batch, HD))
    worst, events = 0.0, []
    for t in range(steps):
        out, reps = kc.decode_step(xs[t][:, None, :], dev, w, cfg)
        y = out.cpu().numpy()[:, 0]
        for b in range(batch):
            yr, rr = refs[b].decode_step(xs[t, b][None], wq, wk, wv, wo, ini)
            worst = max(worst, np.abs(y[b] - yr[0]).max() / max(1.0, np.abs(yr[0]).max()))
            assert bool(reps[b].compression_event) == bool(rr.compression_event), t
            assert reps[b].bytes_after == rr.bytes_after and reps[b].bytes_before == rr.bytes_before, t
            assert reps[b].decompress_flops == rr.decompress_flops, t
        if reps[0].compression_event:
            events.append(t)
    sh = dev.shape()
    for b in range(batch):
        assert sh["n_blocks"] == [refs[b].segment_info(0)[0], refs[b].segment_info(1)[0]]
        assert sh["tail_len"] == [refs[b].segment_info(0)[1], refs[b].segment_info(1)[1]]
    return worst, events, dev, refs


def test_periodic_joint_recompression_matches_reference():
    """Textual keys compressed (key-only), period 4: re-factorisation
    events every 4 steps on both sides; outputs agree within the fp32 bound."""
    worst, events, _, _ = _side_by_side((4, 2, 16), 40, 8, (8, 8, 8, 0), steps=13, period=4, dtype="f32")
    print(f"period 4: events at steps {events}, worst rel err {worst:.2e}")
    assert events == [3, 7, 11]
    assert worst <= 1e-4


def test_separate_epochs_and_tiers_match_reference():
    worst, events, dev, refs = _side_by_side(
        (4, 4, 8), 48, 6, (8, 8, 6, 6), steps=9, period=3, dtype="f64", recompress="separate_epochs",
        tiering=((0.25, 0.5, 0.25), (1.0, 0.5, 0.25), (1.0, 0.75, 0.5)))
    print(f"separate epochs + 3 tiers: events {events}, worst rel err {worst:.2e}, blocks {dev.shape()['n_blocks']}")
    assert len(events) == 3 and dev.shape()["n_blocks"][1] == 4
    assert worst <= 1e-5


def test_600_step_run_with_period_512_matches_reference():
    """The reference default period (512): the textual tail reaches 512 rows at step
    511 and is jointly re-factorised with its prefill block; decoding continues past it."""
    worst, events, dev, _ = _side_by_side((4, 2, 16), 40, 8, (8, 8, 8, 0), steps=600, period=512, dtype="f32",
                                          batch=1)
    print(f"600 steps: events {events}, worst rel err {worst:.2e}")
    assert events == [511]
    assert dev.shape()["tail_len"][1] == 600 - 512
    assert worst <= 1e-4


def test_compress_now_and_full_matrix_match_reference():
    _torch()
    ref = _ref()
    from oracle import cases
    from paper_2603_23914_b200 import cache as kc
    rng = np.random.default_rng(5)
    H, Hkv, D, n, R = 8, 4, 16, 96, 12
    W = Hkv * D
    k = np.stack([cases.planted(n, W, R, rng) for _ in range(2)])
    v = np.stack([cases.planted(n, W, R, rng) for _ in range(2)])
    txt = rng.standard_normal((2, 5, W))
    dev = kc.LayerCacheBatch(H, Hkv, D, batch=2, dtype="f64")
    dev.append_tokens(0, k, v)
    dev.append_tokens(1, txt, txt * 0.5)
    cfg = kc.DecodeConfig(ranks=kc.MatrixRanks(R, R, 0, 0))
    reps = kc.compress_now(dev, cfg)
    assert all(r.compression_event for r in reps)
    for b in range(2):
        c = ref.RefCache(H, Hkv, D, dtype="f64")
        c.append(0, k[b], v[b])
        c.append(1, txt[b], txt[b] * 0.5)
        c.compress_now(cases.decode_ini(ranks=(R, R, 0, 0)))
        for kind, a in ((0, k[b]), (1, v[b])):
            form, left, right, pos = dev.block(b, 0, 0, kind)
            _, rl, rr, rpos = c.block(0, 0, kind)
            assert form == "lowrank" and left.shape == rl.shape
            assert np.array_equal(pos, rpos)
            # reconstructions, never raw factors (SVD signs are ambiguous)
            assert np.abs(left @ right - rl @ rr).max() <= 1e-5 * np.abs(a).max()
            assert np.abs(right @ right.T - np.eye(R)).max() <= 1e-5
    full = kc.segment_full_matrix(dev, 0, 0)
    for b in range(2):
        _, left, right, _ = dev.block(b, 0, 0, 0)
        assert np.allclose(full[b], left @ right, atol=1e-5 * np.abs(full[b]).max())
    full_t = kc.segment_full_matrix(dev, 1, 1)
    assert np.array_equal(full_t, txt * 0.5)
    mb = dev.memory_bytes(0, 2)
    assert mb["visual"] == 2 * 2 * (n * R + R * W) and mb["textual"] == 2 * 2 * 5 * W


def test_error_behaviour():
    torch = _torch()
    from paper_2603_23914_b200 import cache as kc
    dev = kc.LayerCacheBatch(4, 4, 8, batch=1, dtype="f32")
    dev.append_tokens(0, np.ones((4, 32)), np.ones((4, 32)))
    w = kc.AttentionWeights(np.eye(32), np.eye(32), np.eye(32), np.eye(32), dtype="f32")
    cfg = kc.DecodeConfig(ranks=kc.MatrixRanks(2, 2, 0, 0))
    x = np.zeros((1, 1, 32))
    x[0, 0, 3] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        kc.decode_step(x, dev, w, cfg)
    assert dev.shape()["steps_taken"] == 0 and dev.shape()["tail_len"] == [4, 0]  # nothing changed
    with pytest.raises(ValueError, match="alpha"):
        kc.decode_step(np.zeros((1, 1, 32)), dev, w, kc.DecodeConfig(alpha=1.5))
    with pytest.raises(ValueError, match="ratios must sum"):
        kc.decode_step(np.zeros((1, 1, 32)), dev, w,
                       kc.DecodeConfig(tiering=kc.TierSpec([0.5, 0.6], [1.0, 1.0], [1.0, 0.5])))
    with pytest.raises(ValueError, match="model_width"):
        kc.decode_step(np.zeros((1, 1, 31)), dev, w, cfg)
    torch.cuda.synchronize()
