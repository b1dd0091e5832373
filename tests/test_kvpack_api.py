"""The kvpack-compatible Python surface (paper_2603_23914_b200.kvpack), ported
from the reference's binding smoke tests (proj/tests/python/test_smoke.py).
Host accounting is exact; the factorisation runs in fp32 on the GPU, so the
reference's 1e-10 bounds become fp32 bounds (1e-5 relative), stated per test."""
import numpy as np
import pytest

from paper_2603_23914_b200 import kvpack


def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_compression_ratio_closed_form():  # test_smoke.py:15-20
    assert kvpack.compression_ratio(1000, 5120, 64) == pytest.approx(13.071895424836601, abs=1e-12)
    assert kvpack.compression_ratio(16, 128, 8) == pytest.approx(16 * 128 / (16 * 8 + 8 * 128))
    assert kvpack.compression_ratio(100, 64, 0) == 1.0
    with pytest.raises(ValueError):
        kvpack.compression_ratio(0, 64, 4)


def test_flops_reduction_exact():  # test_smoke.py:23-26
    flops, reduction = kvpack.partial_decompress_flops(1000, 5120, [0.1, 0.9], [64, 16])
    assert flops == 212992000
    assert abs(reduction - 0.675) <= 1e-15
    with pytest.raises(ValueError):
        kvpack.partial_decompress_flops(10, 10, [0.5], [4, 2])


def test_truncated_svd_validation():  # linalg.cpp:15-24 (checked before any device work)
    with pytest.raises(ValueError):
        kvpack.truncated_svd(np.ones((4, 3)), 0)
    with pytest.raises(ValueError):
        kvpack.truncated_svd(np.ones((4, 3)), 4)
    with pytest.raises(ValueError):
        kvpack.truncated_svd(np.full((4, 3), np.nan), 2)
    left, right = kvpack.truncated_svd(np.zeros((5, 4)), 2)  # zero matrix: coordinate rows
    assert not left.any() and np.array_equal(right, np.eye(2, 4))


@pytest.mark.gpu
def test_truncated_svd_matches_numpy():  # test_smoke.py:29-39, fp32: 1e-5 relative
    _gpu()
    rng = np.random.default_rng(3)
    a = rng.standard_normal((40, 24))
    left, right = kvpack.truncated_svd(a, 6)
    assert left.shape == (40, 6) and right.shape == (6, 24)
    err = np.linalg.norm(a - left @ right)
    u, s, vt = np.linalg.svd(a, full_matrices=False)
    best = np.linalg.norm(a - (u[:, :6] * s[:6]) @ vt[:6])
    assert abs(err - best) <= 1e-5 * np.linalg.norm(a)
    assert np.allclose(right @ right.T, np.eye(6), atol=1e-5)


@pytest.mark.gpu
def test_truncated_svd_rank_deficient_keeps_orthonormal_rows():
    # rank 5 < requested 8 (linalg.cpp:26-29: zero singular values keep orthonormal right rows):
    # the device Jacobi eigensolver leaves the null components dead, the complement fills them
    _gpu()
    rng = np.random.default_rng(8)
    a = rng.standard_normal((40, 5)) @ rng.standard_normal((5, 24))
    for method in ("exact", "randomized"):
        left, right = kvpack.truncated_svd(a, 8, method=method, seed=2)
        assert np.abs(a - left @ right).max() <= 1e-4 * np.abs(a).max()
        assert np.abs(right @ right.T - np.eye(8)).max() <= 1e-5
        # rank prefix 5 already reconstructs the matrix
        assert np.abs(a - left[:, :5] @ right[:5]).max() <= 1e-4 * np.abs(a).max()


@pytest.mark.gpu
def test_singular_values_graded_spectrum():
    # the one-sided block Jacobi (small_linalg.cu) against LAPACK on a spectrum spanning 1e3 (the
    # fp32 sketch products and CholeskyQR keep ~1e-3 relative accuracy down to ~1e-3 of the top
    # singular value)
    _gpu()
    rng = np.random.default_rng(9)
    u, _ = np.linalg.qr(rng.standard_normal((96, 64)))
    v, _ = np.linalg.qr(rng.standard_normal((80, 64)))
    s = np.logspace(0, -3, 64)
    a = (u * s) @ v.T
    got = kvpack.singular_values(a)
    assert np.allclose(got[:64], s, rtol=2e-3, atol=1e-6 * s[0])
    assert np.all(got[64:] <= 1e-5 * s[0])


@pytest.mark.gpu
def test_randomized_svd_close_to_optimal():  # test_smoke.py:42-50
    _gpu()
    rng = np.random.default_rng(4)
    base = rng.standard_normal((60, 8)) @ rng.standard_normal((8, 30))
    noisy = base + 0.01 * rng.standard_normal((60, 30))
    left, right = kvpack.truncated_svd(noisy, 8, method="randomized", seed=1)
    err = np.linalg.norm(noisy - left @ right)
    s = np.linalg.svd(noisy, compute_uv=False)
    best = float(np.sqrt((s[8:] ** 2).sum()))
    assert err <= 1.5 * best


@pytest.mark.gpu
def test_randomized_svd_tracks_reference_at_tensor_core_shape():
    # The tensor-core range finder (bf16 operands, hi/lo split for the last power
    # iteration and B = Q^T A) against the reference's own randomized SVD
    # (oracle/_ref, linalg.cpp:68-105) on a latent-factor matrix of the bench's
    # kind: reconstruction error within 3% of the reference's, orthonormal rows.
    _gpu()
    from oracle import kvpack_oracle as ko
    from oracle import ref
    T, H, D, R = 1152, 16, 128, 184
    a = ko.latent_factor_matrix(T, H, D, 2 * R, 0.98, R, 1e-2, 21, ko.stream_id(2, 0, 0, 0))
    left, right = kvpack.truncated_svd(a, R, method="randomized", seed=0)
    err = np.linalg.norm(a - left @ right) / np.linalg.norm(a)
    rl, rr = ref.truncated_svd(a, R, method="randomized", seed=0)
    ref_err = np.linalg.norm(a - rl @ rr) / np.linalg.norm(a)
    assert err <= 1.03 * ref_err, (err, ref_err)
    assert np.abs(right @ right.T - np.eye(R)).max() <= 1e-5


@pytest.mark.gpu
def test_variance_helpers():  # test_smoke.py:53-62, fp32 singular values
    _gpu()
    rng = np.random.default_rng(5)
    a = rng.standard_normal((50, 10)) @ np.diag([8.0, 4.0, 2.0, 1.0, 0, 0, 0, 0, 0, 0])
    s = np.linalg.svd(a, compute_uv=False)
    assert np.allclose(kvpack.singular_values(a)[:4], s[:4], rtol=1e-5)
    evr = kvpack.explained_variance_ratio(a, 2)
    assert evr == pytest.approx(float((s[:2] ** 2).sum() / (s ** 2).sum()), abs=1e-6)
    rank, achieved = kvpack.rank_for_variance(a, 0.999, 10)
    assert achieved >= 0.999
    assert kvpack.explained_variance_ratio(a, rank - 1) < 0.999


@pytest.mark.gpu
def test_ema_update_hand_case():  # test_smoke.py:65-69 (bit-exact EMA)
    _gpu()
    scores = kvpack.ema_update(np.array([0.4, 0.0]), np.array([[0.1, 0.9], [0.1, 0.9]]), alpha=0.25)
    assert scores[0] == pytest.approx(0.11875, abs=1e-15)


@pytest.mark.gpu
def test_assign_groups_partition():  # test_smoke.py:72-81
    _gpu()
    masks = kvpack.assign_groups(np.array([0.9, 0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.05, 0.8]), [0.3, 0.3, 0.4],
                                 [16, 8, 4])
    assert [len(m) for m in masks] == [3, 3, 4]
    assert sorted(i for m in masks for i in m) == list(range(10))
    assert 0 in masks[0] and 8 in masks[2]


def test_oracle_quantize_roundtrip_bound():  # test_smoke.py:83-91 against the compiled reference
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(6)
    a = rng.uniform(-2.0, 2.0, size=(128, 16))
    out = ref.quantize_roundtrip(a, 32)
    for j in range(a.shape[1]):
        for g in range(0, a.shape[0], 32):
            block = a[g:g + 32, j]
            assert np.abs(out[g:g + 32, j] - block).max() <= (block.max() - block.min()) / 30.0 + 1e-12


@pytest.mark.gpu
def test_quantize_roundtrip_bit_exact_with_reference():
    # test_smoke.py:83-91 plus edge cases (quantize.cpp:10-54): ragged last group, group_size 1,
    # constant groups (zero scale), +-0 ties, a single row; bit-identical to the compiled reference
    _gpu()
    from oracle import ref
    rng = np.random.default_rng(6)
    a = rng.uniform(-2.0, 2.0, size=(128, 16))
    out = kvpack.quantize_roundtrip(a, group_size=32)
    for j in range(a.shape[1]):
        for g in range(0, a.shape[0], 32):
            block = a[g:g + 32, j]
            assert np.abs(out[g:g + 32, j] - block).max() <= (block.max() - block.min()) / 30.0 + 1e-12
    cases = [(a, 32), (rng.standard_normal((67, 9)), 16), (rng.standard_normal((5, 3)), 1),
             (np.r_[np.full((8, 4), 0.5), rng.standard_normal((9, 4))], 8),
             (np.array([[0.0, -0.0], [-0.0, 0.0], [1.0, -1.0]]), 2), (rng.standard_normal((1, 7)), 64),
             (rng.standard_normal((300, 40)) * 1e3, 64)]
    for m, gs in cases:
        got = kvpack.quantize_roundtrip(m, group_size=gs)
        want = ref.quantize_roundtrip(m, gs)
        assert np.array_equal(got.view(np.int64), want.view(np.int64)), gs
    with pytest.raises(ValueError):
        kvpack.quantize_roundtrip(a, group_size=0)
    with pytest.raises(ValueError):
        kvpack.quantize_roundtrip(np.array([[np.nan]]))
