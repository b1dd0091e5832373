"""GPU parity of the low-level kernels against the reference's golden vectors
(tests/golden, produced by the compiled reference) — through the C-ABI."""
import ctypes as C
import glob
from pathlib import Path

import numpy as np
import pytest

GOLDEN = Path(__file__).resolve().parent / "golden"
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.mark.parametrize("path", sorted(glob.glob(str(GOLDEN / "attend_*.npz"))))
def test_attend_plan_matches_reference(torch_cuda, path):
    from kvp_testlib import attend_on_gpu
    st = dict(np.load(path))
    dtype = str(st["dtype"])
    ctx, ha, hat = attend_on_gpu(st, st["plan"], st["queries"], st["qpos"], dtype=dtype)
    # fp32 caches: the reference rounds rebuilt rows to float before attending;
    # the GPU never rebuilds rows, so the bound is float rounding (1e-4 rel).
    tol = 1e-4 if dtype == "f32" else 1e-10
    scale = max(1.0, float(np.abs(st["context"]).max()))
    assert np.abs(ctx - st["context"]).max() <= tol * scale
    assert np.abs(ha - st["head_avg"]).max() <= tol
    # head_avg scattered to importance-table order (decoder.cpp:595-600)
    tpos = {int(p): i for i, p in enumerate(st["imp_positions"])}
    for j, p in enumerate(st["plan"][:, 5]):
        assert hat[:, tpos[int(p)]] == pytest.approx(ha[:, j], abs=0)
    assert np.allclose(ha.sum(axis=1), 1.0, atol=1e-9)


def test_assign_tiers_bit_exact(torch_cuda):
    from paper_2603_23914_b200 import _capi as capi
    g = dict(np.load(GOLDEN / "importance.npz"))
    for k in range(int(g["n_groups"])):
        s = np.ascontiguousarray(g[f"g{k}_scores"])
        ratios = np.ascontiguousarray(g[f"g{k}_ratios"], dtype=np.float64)
        ranks = np.ascontiguousarray(g[f"g{k}_ranks"], dtype=np.int32)
        out = np.zeros(s.size, dtype=np.uint32)
        capi.call("kvp_assign_groups_host", s.size, s.ctypes.data, ratios.size, ratios.ctypes.data,
                  ranks.ctypes.data, out.ctypes.data)
        assert np.array_equal(out, g[f"g{k}_tier"]), k


def test_ema_bit_exact(torch_cuda):
    from paper_2603_23914_b200 import _capi as capi
    g = dict(np.load(GOLDEN / "importance.npz"))
    for k in range(int(g["n_ema"])):
        s = np.ascontiguousarray(g[f"e{k}_scores"]).copy()
        a = np.ascontiguousarray(g[f"e{k}_attn"])
        capi.call("kvp_update_importance_host", s.size, s.ctypes.data, a.shape[0], a.ctypes.data,
                  float(g[f"e{k}_alpha"]))
        assert np.array_equal(s, g[f"e{k}_out"]), k


def test_ema_rejects_non_distribution(torch_cuda):
    from paper_2603_23914_b200 import _capi as capi
    s = np.array([0.5, 0.5])
    a = np.array([[0.9, 0.3]])
    with pytest.raises(ValueError):
        capi.call("kvp_update_importance_host", 2, s.ctypes.data, 1, a.ctypes.data, 0.25)


def test_assign_tiers_device_batched(torch_cuda):
    """Many tables in one launch, with rank outputs (the engine's form)."""
    torch = torch_cuda
    from oracle import kvpack_oracle as ko
    from paper_2603_23914_b200 import _capi as capi
    rng = np.random.default_rng(5)
    n, tables = 2304, 16
    s = rng.uniform(0, 1, (tables, n))
    s[:, ::7] = 0.125
    ds = torch.as_tensor(s).cuda()
    tier = torch.zeros((tables, n), dtype=torch.uint8, device="cuda")
    rk = torch.zeros((tables, n), dtype=torch.int16, device="cuda")
    rv = torch.zeros((tables, n), dtype=torch.int16, device="cuda")
    ratios = np.array([0.25, 0.75])
    kr = np.array([368, 368], dtype=np.int32)
    vr = np.array([368, 92], dtype=np.int32)
    capi.call("kvp_assign_tiers", tables, n, ds.data_ptr(), n, 2, ratios.ctypes.data, kr.ctypes.data,
              vr.ctypes.data, tier.data_ptr(), rk.data_ptr(), rv.data_ptr(), None)
    torch.cuda.synchronize()
    for t in range(tables):
        want = ko.assign_groups(s[t], [0.25, 0.75], [368, 92])
        assert np.array_equal(tier[t].cpu().numpy(), want)
        assert np.array_equal(rv[t].cpu().numpy(), np.where(want == 0, 368, 92))


@pytest.mark.parametrize("n", [1, 7, 100, 513, 2048, 4096, 5000])
def test_assign_tiers_select_matches_oracle(torch_cuda, n):
    """The radix-select path (n <= 4096) and the sort path (larger n) against the
    reference ordering (importance.cpp:67-117): heavy ties, zeros and -0.0,
    three and four groups, empty groups."""
    torch = torch_cuda
    from oracle import kvpack_oracle as ko
    from paper_2603_23914_b200 import _capi as capi
    rng = np.random.default_rng(n)
    tables = 6
    s = np.round(rng.uniform(0, 1, (tables, n)), 2)  # many exact ties
    s[0] = 0.0
    s[1, ::3] = -0.0
    s[2, : n // 2] = 1e-300
    ds = torch.as_tensor(s).cuda()
    for ratios in ([0.25, 0.75], [0.125, 0.375, 0.5], [0.0, 0.5, 0.0, 0.5], [1.0, 0.0]):
        g = len(ratios)
        ranks = np.array(sorted(rng.integers(1, 64, g), reverse=True), dtype=np.int32)
        tier = torch.zeros((tables, n), dtype=torch.uint8, device="cuda")
        r = np.ascontiguousarray(ratios, dtype=np.float64)
        capi.call("kvp_assign_tiers", tables, n, ds.data_ptr(), n, g, r.ctypes.data, ranks.ctypes.data,
                  ranks.ctypes.data, tier.data_ptr(), None, None, None)
        torch.cuda.synchronize()
        got = tier.cpu().numpy()
        for t in range(tables):
            want = ko.assign_groups(s[t], list(ratios), list(ranks))
            assert np.array_equal(got[t], want), (n, ratios, t)
