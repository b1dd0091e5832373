"""GPU end-to-end parity of the device engine (prefill compaction + decode
steps) against the reference on the same synthetic workload.

The workload is regenerated on the CPU with the oracle's Philox restatement
(harness.cpp:82-173 streams).  Compaction is checked on reconstructions
(SVD signs are ambiguous); decoding is checked against the reference's own
decode_step (oracle/_ref, double precision) fed the engine's bf16 factors, and
against the dense fp64 attention chain, with the bf16 storage bounds of
SURVEY.md §8c."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SPEC = dict(H=4, Hkv=4, D=64, L=2, B=2, n=96, t0=16, steps=4, rank=16, seed=11)
# BASELINE configs[1] (C2) geometry: LLaVA-1.5-7B, 4 x 576 visual + 64 text tokens, rank 368 (1 instance x 2 layers)
SPEC_C2 = dict(H=32, Hkv=32, D=128, L=2, B=1, n=2304, t0=64, steps=2, rank=368, seed=11)


def _torch():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def d2h(ptr, nbytes):
    _torch()
    rt = C.CDLL("libcudart.so.12")
    out = np.empty(nbytes, dtype=np.uint8)
    rc = rt.cudaMemcpy(C.c_void_p(out.ctypes.data), C.c_void_p(ptr), C.c_size_t(nbytes), 2)
    assert rc == 0
    return out


def bf16_to_f64(u16):
    return (np.asarray(u16, dtype=np.uint32) << 16).view(np.float32).astype(np.float64)


def unpack_left(raw_u8, B, n, rank):
    """Inverse of kvp_pack_left: [B][tiles][panels][128 rows][8 swizzled 16-byte chunks]."""
    tiles, panels = (n + 127) // 128, (rank + 63) // 64
    u16 = np.frombuffer(raw_u8.tobytes(), dtype=np.uint16).reshape(B, tiles, panels, 128, 8, 8)
    rows = np.arange(128)
    out = np.empty_like(u16)
    for c in range(8):  # logical chunk c of row r lives at physical chunk c ^ (r % 8)
        out[:, :, :, rows, c, :] = u16[:, :, :, rows, c ^ (rows % 8), :]
    vals = bf16_to_f64(out).reshape(B, tiles, panels, 128, 64)
    return vals.transpose(0, 1, 3, 2, 4).reshape(B, tiles * 128, panels * 64)[:, :n, :rank]


def make_engine(factor_init="compaction", tier=None, s=SPEC):
    from paper_2603_23914_b200.engine import Engine, EngineSpec, ProfileSpec
    vis = ProfileSpec(24, 8, 0.9, 1e-2) if s is SPEC else ProfileSpec(2 * s["rank"], s["rank"], 0.98, 1e-2)
    spec = EngineSpec(heads=s["H"], kv_heads=s["Hkv"], head_dim=s["D"], layers=s["L"], batch=s["B"],
                      visual_tokens=s["n"], textual_tokens=s["t0"], decode_steps=s["steps"], rank_k=s["rank"],
                      rank_v=s["rank"], seed=s["seed"], visual=vis,
                      textual=ProfileSpec(6, 2, 0.9, 1e-3), factor_init=factor_init, svd_seed=3,
                      tier_ratio=tier[0] if tier else 0.0, tier_value_fraction=tier[1] if tier else 1.0)
    eng = Engine(spec)
    eng.prefill()
    return eng


def layer_state(eng, l, s=SPEC):
    from paper_2603_23914_b200 import _capi as capi
    W, HD = s["Hkv"] * s["D"], s["H"] * s["D"]
    cap = s["t0"] + s["steps"]
    v = eng.layer(l)
    pk = capi.lib().kvp_packed_left_bytes(s["B"], s["n"], s["rank"])
    st = {"n_tail": v.n_tail}
    st["left_k"] = unpack_left(d2h(v.left_k, pk), s["B"], s["n"], s["rank"])
    st["left_v"] = unpack_left(d2h(v.left_v, pk), s["B"], s["n"], s["rank"])
    nr = s["B"] * s["rank"] * W * 2
    st["right_k"] = bf16_to_f64(d2h(v.right_k, nr).view(np.uint16)).reshape(s["B"], s["rank"], W)
    st["right_v"] = bf16_to_f64(d2h(v.right_v, nr).view(np.uint16)).reshape(s["B"], s["rank"], W)
    nt = s["B"] * cap * W * 2
    st["tail_k"] = bf16_to_f64(d2h(v.tail_k, nt).view(np.uint16)).reshape(s["B"], cap, W)
    st["tail_v"] = bf16_to_f64(d2h(v.tail_v, nt).view(np.uint16)).reshape(s["B"], cap, W)
    st["imp"] = d2h(v.importance, s["B"] * (s["n"] + cap) * 8).view(np.float64).reshape(s["B"], s["n"] + cap)
    st["wqkv"] = bf16_to_f64(d2h(v.w_qkv, HD * (HD + 2 * W) * 2).view(np.uint16)).reshape(HD, HD + 2 * W)
    st["wo"] = bf16_to_f64(d2h(v.w_o, HD * HD * 2).view(np.uint16)).reshape(HD, HD)
    return st


def test_compaction_reconstructs_visual_segments():
    from oracle import kvpack_oracle as ko
    from oracle import ref
    eng = make_engine()
    s = SPEC
    for l in range(s["L"]):
        st = layer_state(eng, l)
        for kind, kn in ((0, "k"), (1, "v")):
            for b in range(s["B"]):
                a = ko.latent_factor_matrix(s["n"], s["Hkv"], s["D"], 24, 0.9, 8, 1e-2, s["seed"],
                                            ko.stream_id(2, b, l, kind))
                rec = st[f"left_{kn}"][b] @ st[f"right_{kn}"][b]
                err = np.linalg.norm(a - rec) / np.linalg.norm(a)
                # the reference's own randomized SVD (oracle/_ref) on the same matrix
                rl, rr = ref.truncated_svd(a, s["rank"], method="randomized", seed=3)
                ref_err = np.linalg.norm(a - rl @ rr) / np.linalg.norm(a)
                assert err <= 1.05 * ref_err, (l, kn, b, err, ref_err)
                gram = st[f"right_{kn}"][b] @ st[f"right_{kn}"][b].T
                assert np.abs(gram - np.eye(s["rank"])).max() <= 2e-2
        # weights follow the reference's streams (harness.cpp:138-151)
        HD, W = s["H"] * s["D"], s["Hkv"] * s["D"]
        wq = ko.gaussian_matrix(HD, HD, s["seed"], ko.stream_id(1, 0, l, 0)) / np.sqrt(HD)
        assert np.abs(st["wqkv"][:, :HD] - wq).max() <= 4e-3 * np.abs(wq).max()
    eng.close()


CASES = [("small", SPEC, None), ("small", SPEC, (0.5, 0.25)), ("c2", SPEC_C2, None)]


@pytest.mark.parametrize("name,s,tier", CASES, ids=["untiered", "two_tier", "c2_geometry"])
def test_decode_steps_match_reference(name, s, tier):
    """Engine decode vs the reference decode_step (double) on the engine's own
    bf16 factors and weights, layer by layer, every instance: untiered, with
    two-tier attention-aware value decompression (the reference's [decode.tiering]:
    half the tokens by importance at full rank, the rest at a quarter of the value
    rank), and at the C2 geometry (BASELINE configs[1]).  The engine rounds the
    activations to bf16 before each projection and keeps the new K/V rows in bf16;
    the reference chain stays fp64 — the bound is the bf16 storage bound."""
    torch = _torch()
    from oracle import ref
    from oracle.cases import decode_ini
    H, Hkv, D, L, B = s["H"], s["Hkv"], s["D"], s["L"], s["B"]
    W, HD = Hkv * D, H * D
    eng = make_engine(tier=tier, s=s)
    states = [layer_state(eng, l, s) for l in range(L)]
    tiering = ((tier[0], 1.0 - tier[0]), (1.0, 1.0), (1.0, tier[1])) if tier else None
    ini = decode_ini(ranks=(s["rank"], s["rank"], 0, 0), tiering=tiering, period=None, alpha=0.25)
    # reference caches holding the engine's factors as their joint visual block, textual tail verbatim
    caches = {}
    for l in range(L):
        for b in range(B):
            c = ref.RefCache(H, Hkv, D, dtype="f64")
            st = states[l]
            c.append(0, np.zeros((s["n"], W)), np.zeros((s["n"], W)))
            c.factor_tail(0, (st["left_k"][b], st["right_k"][b]), (st["left_v"][b], st["right_v"][b]))
            c.append(1, st["tail_k"][b, :s["t0"]], st["tail_v"][b, :s["t0"]])
            caches[(l, b)] = c
    rng = np.random.default_rng(7)
    xs = rng.standard_normal((s["steps"], B, HD)).astype(np.float32)
    xd = torch.empty((B, HD), dtype=torch.float32, device="cuda")
    yd = torch.empty((B, HD), dtype=torch.float32, device="cuda")
    worst = 0.0
    for t in range(s["steps"]):
        if tier:
            # tier membership is a discontinuous function of the importance ranking: hand the reference the
            # engine's pre-step importance (fp32 head averages vs fp64 can swap near-tied tokens across the
            # group boundary), so the comparison measures the arithmetic; the importance itself is checked below
            for l in range(L):
                imp = layer_state(eng, l, s)["imp"]
                for b in range(B):
                    n_tab = len(caches[(l, b)].importance()[1])
                    caches[(l, b)].set_importance(imp[b, :n_tab])
        xd.copy_(torch.from_numpy(xs[t]))
        eng.step(xd.data_ptr(), yd.data_ptr(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        y = yd.cpu().numpy().astype(np.float64)
        for b in range(B):
            h = xs[t, b].astype(np.float64)
            for l in range(L):
                st = states[l]
                wq, wk, wv = st["wqkv"][:, :HD], st["wqkv"][:, HD:HD + W], st["wqkv"][:, HD + W:]
                h, _ = caches[(l, b)].decode_step(h[None, :], wq, wk, wv, st["wo"], ini)
                h = h[0]
            rel = np.linalg.norm(y[b] - h) / np.linalg.norm(h)
            worst = max(worst, rel)
    print(f"{name} tier={tier}: worst relative output error {worst:.3e} over {s['steps']} steps")
    # bf16 activations into the projection GEMMs, bf16 K/V rows and context vs the fp64 reference chain
    assert worst <= 3e-2, worst
    # bookkeeping: the tail grew by one row per step, new tokens' importance was updated
    st = layer_state(eng, 0, s)
    assert st["n_tail"] == s["t0"] + s["steps"]
    pos, sc = caches[(0, 0)].importance()
    assert np.abs(st["imp"][0, :len(sc)] - sc).max() <= 2e-2
    eng.close()
