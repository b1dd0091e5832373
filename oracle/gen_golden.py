"""ORACLE / TEST INFRASTRUCTURE ONLY — writes tests/golden/*.npz.

Golden vectors produced by the reference itself (its own C++ sources compiled
by oracle/Makefile into oracle/_ref/libkvpack_ref.so, driven through
oracle/ref.py).  Run in the build container (needs /root/reference to build
the library):

    make -C oracle && python -m oracle.gen_golden

The fixtures pin the numpy restatement (oracle/kvpack_oracle.py) and are the
inputs/outputs the GPU parity tests replay through the product C-ABI.
"""
from __future__ import annotations

from pathlib import Path

import numpy as np

from . import cases, ref
from . import kvpack_oracle as ko

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def gen_rng():
    streams = [(0, 0), (42, 1), (0x0123456789ABCDEF, 0xFEDCBA9876543210), (7, ko.SVD_STREAM)]
    g = {f"gauss_{i}": ref.gaussian_matrix(1, 257, s, t)[0] for i, (s, t) in enumerate(streams)}
    g["streams"] = np.array(streams, dtype=np.uint64)
    g["lfm"] = ref.latent_factor_matrix(12, 2, 2, 4, 6, 0.9, 3, 0.01, 5, ko.stream_id(2, 1, 3, 0))
    g["lfm_args"] = np.array([12, 2, 2, 4, 6, 3, 5, ko.stream_id(2, 1, 3, 0)], dtype=np.uint64)
    np.savez_compressed(OUT / "rng.npz", **g)


def gen_importance():
    rng = np.random.default_rng(1234)
    d = {}
    specs = [([0.25, 0.75], [16, 8]), ([0.3, 0.3, 0.4], [32, 16, 8]), ([0.125, 0.875], [128, 128]),
             ([0.5, 0.25, 0.25], [64, 16, 4]), ([1.0], [8])]
    k = 0
    for n in (1, 2, 10, 33, 257, 1000, 4096):
        for ratios, ranks in specs:
            s = rng.uniform(0, 1, n)
            if n > 4:  # ties + exact zeros + quantised values
                s[rng.integers(0, n, n // 3)] = 0.25
                s[rng.integers(0, n, n // 7)] = 0.0
                s[: n // 5] = np.round(s[: n // 5], 2)
            d[f"g{k}_scores"] = s
            d[f"g{k}_ratios"] = np.array(ratios)
            d[f"g{k}_ranks"] = np.array(ranks, dtype=np.uint64)
            d[f"g{k}_tier"] = ref.assign_groups(s, ratios, ranks)
            k += 1
    d["n_groups"] = np.array(k)
    k = 0
    for n, tq, alpha in ((2, 1, 0.25), (16, 2, 0.3), (300, 1, 0.25), (300, 3, 0.0), (300, 2, 1.0),
                         (4161, 1, 0.25)):
        s = rng.uniform(0, 1, n)
        a = rng.uniform(0.01, 1, (tq, n))
        a /= a.sum(axis=1, keepdims=True)
        d[f"e{k}_scores"], d[f"e{k}_attn"], d[f"e{k}_alpha"] = s, a, np.array(alpha)
        d[f"e{k}_out"] = ref.update_importance(s, a, alpha)
        k += 1
    d["n_ema"] = np.array(k)
    np.savez_compressed(OUT / "importance.npz", **d)


ATTEND_SPECS = [
    # name, kwargs
    ("mha", dict(seed=11, geom=(4, 4, 8), n_vis=40, n_txt=6, rank=8, tq=2)),
    ("gqa", dict(seed=21, geom=(8, 2, 8), n_vis=30, n_txt=5, rank=6, tq=3)),
    ("tiers3", dict(seed=31, geom=(4, 4, 8), n_vis=32, n_txt=0, rank=16, tq=1,
                    tiering=([0.25, 0.5, 0.25], [1.0, 0.5, 0.125], [1.0, 0.25, 0.125]))),
    ("tiers2_f32", dict(seed=41, geom=(4, 4, 16), n_vis=64, n_txt=9, rank=12, tq=1, dtype="f32",
                        tiering=([0.375, 0.625], [1.0, 1.0], [1.0, 0.25]))),
    ("hot", dict(seed=51, geom=(4, 4, 8), n_vis=37, n_txt=4, rank=8, tq=2, scale_q=50.0)),
    ("keyonly", dict(seed=61, geom=(4, 4, 8), n_vis=24, n_txt=3, rank=6, tq=1, ranks=(6, 0, 0, 0))),
    ("c1_like", dict(seed=71, geom=(8, 8, 16), n_vis=72, n_txt=8, rank=4, tq=1, dtype="f32",
                     planted_rank=False)),
]

DECODE_SPECS = [
    ("plain", dict(seed=101, geom=(4, 4, 8), n_vis=48, n_txt=8, rank=8, steps=5)),
    ("gqa_tiers", dict(seed=111, geom=(8, 2, 8), n_vis=40, n_txt=6, rank=8, steps=4,
                       tiering=([0.25, 0.75], [1.0, 0.5], [1.0, 0.25]))),
    ("f32", dict(seed=121, geom=(4, 4, 8), n_vis=48, n_txt=8, rank=8, steps=4, dtype="f32")),
]


def gen_attend():
    for name, kw in ATTEND_SPECS:
        np.savez_compressed(OUT / f"attend_{name}.npz", **cases.attend_case(**kw))
    for name, kw in DECODE_SPECS:
        np.savez_compressed(OUT / f"decode_{name}.npz", **cases.decode_case(**kw))


def gen_svd():
    rng = np.random.default_rng(77)
    d = {}
    mats = [("gauss", rng.standard_normal((40, 24)), 6), ("planted", cases.planted(60, 32, 5, rng), 5),
            ("wide", rng.standard_normal((20, 50)), 7),
            ("noisy", cases.planted(80, 48, 12, rng, 0.6) + 0.01 * rng.standard_normal((80, 48)), 8)]
    for i, (name, a, r) in enumerate(mats):
        for method in ("exact", "randomized"):
            left, right = ref.truncated_svd(a, r, method=method, seed=7)
            d[f"{name}_a"] = a
            d[f"{name}_rank"] = np.array(r)
            d[f"{name}_{method}_err"] = np.array(np.linalg.norm(a - left @ right))
        d[f"{name}_sv"] = ref.singular_values(a)
    d["names"] = np.array([m[0] for m in mats])
    np.savez_compressed(OUT / "svd.npz", **d)


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    gen_rng()
    gen_importance()
    gen_attend()
    gen_svd()
    print("golden fixtures ->", OUT)


if __name__ == "__main__":
    main()
