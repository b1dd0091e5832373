"""KVPK snapshots (snapshot.hpp:12-49, snapshot.cpp:251-371) of device caches.

CPU: the reference's own save_cache writes a file, our parser reads every field back.
GPU: device cache -> our save_cache -> the reference's load_cache (and back) at widths 2/4/8,
plus a decode step from the loaded device cache against the reference decode_step."""
import numpy as np
import pytest

from oracle import cases, ref

pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


def _ref_cache(seed=3, H=4, Hkv=2, D=16, n=40, nt=6, ranks=(5, 4, 0, 0)):
    rng = np.random.default_rng(seed)
    W = Hkv * D
    c = ref.RefCache(H, Hkv, D, layer=7)
    c.append(0, cases.planted(n, W, 6, rng), cases.planted(n, W, 6, rng))
    c.append(1, rng.standard_normal((nt, W)), rng.standard_normal((nt, W)))
    c.compress_now(cases.decode_ini(ranks=ranks))
    c.append(1, rng.standard_normal((3, W)), rng.standard_normal((3, W)))
    pos, _ = c.importance()
    c.set_importance(rng.random(pos.size))
    return c


@pytest.mark.parametrize("width", [2, 4, 8])
def test_reader_parses_reference_snapshot(tmp_path, width):
    from paper_2603_23914_b200.snapshot import read_snapshot
    c = _ref_cache()
    path = str(tmp_path / "a.kvpk")
    c.save(path, width)
    s = read_snapshot(path)
    assert (s["H"], s["Hkv"], s["D"], s["width"], s["layer_index"]) == (4, 2, 16, width, 7)
    tol = {2: 2e-3, 4: 1e-6, 8: 0.0}[width]
    for m in (0, 1):
        nb, tl, _ = c.segment_info(m)
        seg = s["segments"][m]
        k, v, tpos = c.tail(m)
        assert np.array_equal(seg["tail_positions"], tpos)
        assert np.allclose(seg["tail_k"], k, rtol=tol, atol=tol) and np.allclose(seg["tail_v"], v, rtol=tol, atol=tol)
        if nb:
            for kind in (0, 1):
                form, a, b, p = c.block(m, 0, kind)
                assert np.array_equal(seg["compressed_positions"], p)
                assert seg["stores"][kind][0] == form
                assert np.allclose(seg["stores"][kind][1], a, rtol=tol, atol=tol * np.abs(a).max())
    pos, sc = c.importance()
    assert np.array_equal(s["imp_positions"], pos) and np.array_equal(s["imp_scores"], sc)  # f64 always
    assert s["alpha"] == 0.25


def test_reader_rejects_bad_files(tmp_path):
    from paper_2603_23914_b200.snapshot import read_snapshot
    p = tmp_path / "bad.kvpk"
    p.write_bytes(b"NOPE" + bytes(40))
    with pytest.raises(ValueError, match="not a KVPK"):
        read_snapshot(str(p))
    c = _ref_cache()
    good = str(tmp_path / "g.kvpk")
    c.save(good, 4)
    data = open(good, "rb").read()
    (tmp_path / "t.kvpk").write_bytes(data[:len(data) // 2])
    with pytest.raises(ValueError, match="truncated"):
        read_snapshot(str(tmp_path / "t.kvpk"))
    with pytest.raises(OSError):
        read_snapshot(str(tmp_path / "missing.kvpk"))


@pytest.mark.gpu
@pytest.mark.parametrize("width", [2, 4, 8])
def test_device_cache_round_trips_through_reference(tmp_path, width):
    from paper_2603_23914_b200.cache import LayerCacheBatch
    from paper_2603_23914_b200.snapshot import load_cache, save_cache
    rc = _ref_cache(seed=5)
    dev = LayerCacheBatch.from_state([cases.export_state(rc)])
    dev.layer_index = 7
    mine = str(tmp_path / "mine.kvpk")
    save_cache(dev, 0, mine, width)
    # the reference reads our file and holds the same cache (to the payload width)
    back = ref.RefCache.load(mine, 4, 2, 16)
    tol = {2: 2e-3, 4: 1e-6, 8: 0.0}[width]
    for m in (0, 1):
        assert back.segment_info(m)[:2] == rc.segment_info(m)[:2]
        k, v, p = back.tail(m)
        rk, rv, rp = rc.tail(m)
        assert np.array_equal(p, rp) and np.allclose(k, rk, rtol=tol, atol=tol)
        if rc.segment_info(m)[0]:
            for kind in (0, 1):
                f1, a1, b1, p1 = back.block(m, 0, kind)
                f0, a0, b0, p0 = rc.block(m, 0, kind)
                assert f1 == f0 and np.array_equal(p1, p0)
                assert np.allclose(a1, a0, rtol=tol, atol=tol * np.abs(a0).max())
    assert np.array_equal(back.importance()[1], rc.importance()[1])
    # and our loader reads the reference's file into a device cache
    theirs = str(tmp_path / "ref.kvpk")
    rc.save(theirs, width)
    d2 = load_cache(theirs)
    assert d2.shape() == dev.shape()
    for m in (0, 1):
        assert np.allclose(d2.tail(0, m)[0], dev.tail(0, m)[0], rtol=tol, atol=tol)
    assert np.array_equal(d2.importance()[1], dev.importance()[1])


@pytest.mark.gpu
def test_loaded_device_cache_decodes_like_reference(tmp_path):
    from paper_2603_23914_b200.cache import AttentionWeights, DecodeConfig, decode_step
    from paper_2603_23914_b200.snapshot import load_cache
    rc = _ref_cache(seed=9)
    path = str(tmp_path / "s.kvpk")
    rc.save(path, 8)
    dev = load_cache([path, path])  # a batch of two instances from one snapshot
    rng = np.random.default_rng(2)
    HD, W = 64, 32
    ws = [rng.standard_normal(s) / 8 for s in ((HD, HD), (HD, W), (HD, W), (HD, HD))]
    x = rng.standard_normal((1, HD))
    ini = cases.decode_ini(ranks=(5, 4, 0, 0))
    want, _ = rc.decode_step(x, *ws, decode_ini=ini)
    steps0 = dev.shape()["steps_taken"]
    got, _ = decode_step(np.stack([x, x]), dev, AttentionWeights(*ws), DecodeConfig.from_ini(ini))
    got = got.cpu().numpy()
    assert np.abs(got[0] - want).max() <= 1e-9 * max(1.0, np.abs(want).max())
    assert np.array_equal(got[0], got[1])
    assert dev.shape()["steps_taken"] == steps0 + 1
