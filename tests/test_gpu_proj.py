"""Hand-written projection GEMM (kvp_matmul_packed, the decode step's q/k/v and W_o products,
decoder.cpp:574-576, 590) against a plain PyTorch fp32 product of the same bf16 operands."""
import pytest
import torch

from paper_2603_23914_b200 import _capi as capi

pytestmark = pytest.mark.gpu


def run(x, w, out_bf16, ldo=None, reps=1):
    B, K = x.shape
    N = w.shape[1]
    ldo = ldo or N
    pk = torch.empty(capi.lib().kvp_packed_weight_bytes(K, N), dtype=torch.uint8, device="cuda")
    capi.call("kvp_pack_weight", w.data_ptr(), K, N, pk.data_ptr(), None)
    ws = torch.zeros(capi.lib().kvp_matmul_packed_workspace(K, N, B), dtype=torch.uint8, device="cuda")
    out = torch.full((B, ldo), 7.0, dtype=torch.bfloat16 if out_bf16 else torch.float32, device="cuda")
    outs = []
    for _ in range(reps):
        capi.call("kvp_matmul_packed", x.data_ptr(), B, K, pk.data_ptr(), N, out.data_ptr(), ldo, int(out_bf16),
                  ws.data_ptr(), None)
        torch.cuda.synchronize()
        outs.append(out.clone())
    return outs


@pytest.mark.parametrize("B,K,N", [(16, 4096, 12288), (16, 4096, 4096), (64, 5120, 15360), (32, 4096, 12288),
                                   (1, 512, 384), (5, 264, 200), (33, 1024, 640), (200, 256, 1024)])
def test_matmul_packed_matches_fp32(B, K, N):
    g = torch.Generator(device="cuda").manual_seed(B * 7 + K + N)
    x = torch.randn(B, K, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(K, N, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    ref = x.float() @ w.float()
    (y,) = run(x, w, False)
    err = ((y - ref).abs().max() / ref.abs().max()).item()
    assert err <= 1e-5, err
    (yb,) = run(x, w, True)
    errb = ((yb.float() - ref).abs().max() / ref.abs().max()).item()
    assert errb <= 8e-3, errb


def test_matmul_packed_is_deterministic_and_relaunchable():
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(16, 4096, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(4096, 4096, device="cuda", generator=g) / 64).to(torch.bfloat16)
    outs = run(x, w, False, reps=4)
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


def test_matmul_packed_output_stride_untouched_padding():
    g = torch.Generator(device="cuda").manual_seed(4)
    x = torch.randn(8, 1024, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(1024, 512, device="cuda", generator=g) / 32).to(torch.bfloat16)
    (y,) = run(x, w, False, ldo=600)
    assert torch.all(y[:, 512:] == 7.0)
    ref = x.float() @ w.float()
    assert ((y[:, :512] - ref).abs().max() / ref.abs().max()).item() <= 1e-5


def test_matmul_packed_rejects_bad_shapes():
    with pytest.raises(ValueError):
        capi.call("kvp_matmul_packed", 1, 300, 64, 1, 64, 1, 64, 0, 1, None)  # B > 256
    with pytest.raises(ValueError):
        capi.call("kvp_matmul_packed", 1, 4, 64, 1, 64, 1, 32, 0, 1, None)  # ldo < N
