"""KVPK snapshot I/O for device caches (snapshot.hpp:12-49, snapshot.cpp:251-371).

``save_cache(cache, instance, path, scalar_width)`` writes one instance of a device
``LayerCacheBatch`` in the reference's KVPK version-1 layout, so the reference's
``load_cache`` reads it; ``load_cache(paths)`` rebuilds a device ``LayerCacheBatch``
from one or more snapshots of identical structure (one instance each).  The payloads
move through the C-ABI (``kvp_cache_block_get`` / ``kvp_cache_tail_get`` down,
``kvp_cache_append`` / ``kvp_cache_factor_tail`` / ``kvp_cache_set_importance`` /
``kvp_cache_set_counters`` up); the byte layout is host code, like the reference's.

Layout (little-endian): magic "KVPK" | u32 version | u32 H | u32 H_kv | u32 D |
u8 scalar_width | u32 layer_index | u64 next_position | u64 steps_taken | u8 segment
count (2); per segment: u8 modality | u64 T_uc | u64 T_cc | u32 R_k | u32 R_v |
u64 compressed positions | u64 tail positions | tail_k | tail_v | (T_cc > 0) K then
V store: u8 tag (0 plain factors: left, right; 2 dense rows); importance: f64 alpha |
u64 count | (u64 position, f64 score) pairs.  Width-2 payloads are IEEE binary16
(round to nearest even from float, snapshot.cpp:15-45 / :131-145).

Errors follow the reference: bad widths and multi-block (separate-epochs) segments are
parameter errors (``ValueError``), malformed files data errors (``ValueError``), missing
files io errors (``OSError``).  The device cache has no quantized stores, so snapshots
holding quantized payloads (tags 1 and 3) are rejected with ``ValueError``.
"""
from __future__ import annotations

import struct

import numpy as np

from .cache import KEY, TEXTUAL, VALUE, VISUAL, LayerCacheBatch

MAGIC = b"KVPK"
VERSION = 1
_PLAIN_FACTORS, _QUANT_FACTORS, _PLAIN_DENSE, _QUANT_DENSE = 0, 1, 2, 3
_WIDTH_DT = {2: np.float16, 4: np.float32, 8: np.float64}


def _scalars(a: np.ndarray, width: int) -> bytes:
    x = np.ascontiguousarray(a, dtype=np.float64)
    if width == 2:  # float_to_half(static_cast<float>(v)): round to float, then to binary16 (RNE)
        return x.astype(np.float32).astype("<f2").tobytes()
    return x.astype("<f4" if width == 4 else "<f8").tobytes()


def save_cache(cache: LayerCacheBatch, instance: int, path: str, scalar_width: int | None = None,
               alpha: float = 0.25) -> None:
    """save_cache (snapshot.cpp:251-307) of instance `instance` of a device cache."""
    if scalar_width is None:
        scalar_width = {"f64": 8, "f32": 4, "bf16": 4}[cache.dtype]  # bf16 is exact in a float payload
    if scalar_width not in (2, 4, 8):
        raise ValueError("save_cache: scalar width must be 2, 4, or 8")
    if not 0 <= instance < cache.batch:
        raise ValueError("save_cache: instance out of range")
    sh = cache.shape()
    if max(sh["n_blocks"]) > 1:
        raise ValueError("save_cache: KVPK v1 stores one block per segment; consolidate the "
                         "separate-epochs cache first")
    out = [MAGIC, struct.pack("<IIIIBIQQB", VERSION, cache.H, cache.Hkv, cache.D, scalar_width,
                              cache.layer_index, sh["next_position"], sh["steps_taken"], 2)]
    for seg in (VISUAL, TEXTUAL):
        tk, tv, tpos = cache.tail(instance, seg)
        stores, cpos = [], np.zeros(0, dtype=np.uint64)
        if sh["n_blocks"][seg]:
            for kind in (KEY, VALUE):
                form, left, right, pos = cache.block(instance, seg, 0, kind)
                stores.append((form, left, right))
                cpos = pos
        t_cc = int(cpos.size)
        r_k = stores[0][1].shape[1] if stores and stores[0][0] == "lowrank" else 0
        r_v = stores[1][1].shape[1] if stores and stores[1][0] == "lowrank" else 0
        out.append(struct.pack("<BQQII", seg, tk.shape[0], t_cc, r_k, r_v))
        out.append(np.ascontiguousarray(cpos, dtype="<u8").tobytes())
        out.append(np.ascontiguousarray(tpos, dtype="<u8").tobytes())
        out += [_scalars(tk, scalar_width), _scalars(tv, scalar_width)]
        if t_cc:
            for form, left, right in stores:
                if form == "lowrank":
                    out += [struct.pack("<B", _PLAIN_FACTORS), _scalars(left, scalar_width),
                            _scalars(right, scalar_width)]
                else:
                    out += [struct.pack("<B", _PLAIN_DENSE), _scalars(left, scalar_width)]
    pos, scores = cache.importance()
    out.append(struct.pack("<dQ", float(alpha), pos.size))
    rec = np.zeros(pos.size, dtype=[("p", "<u8"), ("s", "<f8")])
    rec["p"], rec["s"] = pos, scores[instance]
    out.append(rec.tobytes())
    with open(path, "wb") as f:
        f.write(b"".join(out))


class _Reader:
    def __init__(self, path: str):
        with open(path, "rb") as f:  # OSError for a missing file, as the reference's io_error
            self.b = f.read()
        self.o = 0

    def take(self, n: int) -> bytes:
        if self.o + n > len(self.b):
            raise ValueError("snapshot: truncated file")
        s = self.b[self.o:self.o + n]
        self.o += n
        return s

    def pod(self, fmt: str):
        v = struct.unpack("<" + fmt, self.take(struct.calcsize("<" + fmt)))
        return v if len(v) > 1 else v[0]

    def array(self, count: int, dt) -> np.ndarray:
        dt = np.dtype(dt).newbyteorder("<")
        return np.frombuffer(self.take(count * dt.itemsize), dtype=dt).astype(np.float64 if dt.kind == "f" else dt)


def read_snapshot(path: str) -> dict:
    """Parse a KVPK v1 file (snapshot.cpp:309-371) into host arrays."""
    r = _Reader(path)
    if r.take(4) != MAGIC:
        raise ValueError(f"not a KVPK snapshot: {path}")
    version = r.pod("I")
    if version != VERSION:
        raise ValueError(f"unsupported KVPK version {version}")
    H, Hkv, D = r.pod("III")
    if H < 1 or Hkv < 1 or D < 1 or H % Hkv:
        raise ValueError("HeadGeometry: heads must be positive and a multiple of kv_heads")
    width = r.pod("B")
    if width not in (2, 4, 8):
        raise ValueError(f"snapshot: bad scalar width {width}")
    layer, next_pos, steps, nseg = r.pod("IQQB")
    if nseg != 2:
        raise ValueError("snapshot: expected 2 segment records")
    W, dt = Hkv * D, _WIDTH_DT[width]
    snap = dict(H=H, Hkv=Hkv, D=D, width=width, layer_index=layer, next_position=next_pos, steps_taken=steps,
                segments={})
    for _ in range(2):
        mod, t_uc, t_cc, r_k, r_v = r.pod("BQQII")
        if mod > 1:
            raise ValueError("snapshot: bad modality tag")
        seg = dict(compressed_positions=r.array(t_cc, np.uint64), tail_positions=r.array(t_uc, np.uint64))
        seg["tail_k"] = r.array(t_uc * W, dt).reshape(t_uc, W)
        seg["tail_v"] = r.array(t_uc * W, dt).reshape(t_uc, W)
        seg["stores"] = []
        if t_cc:
            for rank in (r_k, r_v):
                tag = r.pod("B")
                if tag == _PLAIN_FACTORS:
                    left = r.array(t_cc * rank, dt).reshape(t_cc, rank)
                    seg["stores"].append(("lowrank", left, r.array(rank * W, dt).reshape(rank, W)))
                elif tag == _PLAIN_DENSE:
                    seg["stores"].append(("dense", r.array(t_cc * W, dt).reshape(t_cc, W), None))
                elif tag in (_QUANT_FACTORS, _QUANT_DENSE):
                    raise ValueError("load_cache: quantized stores are not supported by the device cache")
                else:
                    raise ValueError(f"snapshot: unknown payload tag {tag}")
        snap["segments"][mod] = seg
    snap["alpha"] = r.pod("d")
    count = r.pod("Q")
    rec = np.frombuffer(r.take(count * 16), dtype=[("p", "<u8"), ("s", "<f8")])
    snap["imp_positions"], snap["imp_scores"] = rec["p"].astype(np.uint64), rec["s"].astype(np.float64)
    return snap


def load_cache(paths, dtype: str = "f64") -> LayerCacheBatch:
    """load_cache (snapshot.cpp:309-371) into a device cache: one instance per snapshot;
    every snapshot must share the segment structure (counts, ranks, positions)."""
    if isinstance(paths, str):
        paths = [paths]
    snaps = [read_snapshot(p) for p in paths]
    s0 = snaps[0]
    for s in snaps[1:]:
        same = all(s[k] == s0[k] for k in ("H", "Hkv", "D", "layer_index", "next_position", "steps_taken"))
        for m in (0, 1):
            a, b = s["segments"][m], s0["segments"][m]
            same = same and np.array_equal(a["compressed_positions"], b["compressed_positions"]) and \
                np.array_equal(a["tail_positions"], b["tail_positions"]) and \
                [(f, x.shape) for f, x, _ in a["stores"]] == [(f, x.shape) for f, x, _ in b["stores"]]
        if not same or not np.array_equal(s["imp_positions"], s0["imp_positions"]):
            raise ValueError("load_cache: a batch needs snapshots of identical structure")
    c = LayerCacheBatch(s0["H"], s0["Hkv"], s0["D"], batch=len(snaps), dtype=dtype, layer_index=s0["layer_index"])
    W = c.W
    # the device cache assigns positions in append order: replay the runs (blocks, tails) in
    # position order and check that they come out at the recorded positions
    runs = []
    for m in (0, 1):
        seg = s0["segments"][m]
        if seg["compressed_positions"].size:
            runs.append((int(seg["compressed_positions"][0]), m, "block"))
        if seg["tail_positions"].size:
            runs.append((int(seg["tail_positions"][0]), m, "tail"))
    for _, m, what in sorted(runs):
        segs = [s["segments"][m] for s in snaps]
        if what == "tail":
            c.append_tokens(m, np.stack([g["tail_k"] for g in segs]), np.stack([g["tail_v"] for g in segs]))
            continue
        n = segs[0]["compressed_positions"].size
        rows, facs = [], []
        for kind in (KEY, VALUE):
            form = segs[0]["stores"][kind][0]
            if form == "lowrank":
                facs.append((np.stack([g["stores"][kind][1] for g in segs]), np.stack([g["stores"][kind][2] for g in segs])))
                rows.append(np.zeros((len(snaps), n, W)))
            else:
                facs.append(None)
                rows.append(np.stack([g["stores"][kind][1] for g in segs]))
        c.append_tokens(m, rows[0], rows[1])
        c.factor_tail(m, facs[0], facs[1])
    for m in (0, 1):
        want = s0["segments"][m]
        got = [c.block(0, m, 0, KEY)[3]] if c.shape()["n_blocks"][m] else []
        got_c = got[0] if got else np.zeros(0, dtype=np.uint64)
        if not np.array_equal(got_c, want["compressed_positions"]) or \
                not np.array_equal(c.tail(0, m)[2], want["tail_positions"]):
            raise ValueError("load_cache: positions are not consecutive runs (the device cache cannot hold gaps)")
    pos, _ = c.importance()
    if not np.array_equal(pos, s0["imp_positions"]):
        raise ValueError("load_cache: importance positions do not match the payload positions")
    c.set_importance(np.stack([s["imp_scores"] for s in snaps]))
    from . import _capi as capi
    capi.call("kvp_cache_set_counters", c._h, s0["next_position"], s0["steps_taken"])
    return c
