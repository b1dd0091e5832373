"""ORACLE / TEST INFRASTRUCTURE ONLY — a CPU restatement of the reference path.

numpy restatement of the AttentionPack ``kvpack`` reference for the hot path
named by BASELINE.json's north_star.  Every function cites the reference
file:line it follows (``/root/reference/proj/...``).  It is *pinned*: the
tests check it against golden vectors produced by the reference itself
(``tests/golden/*.npz``, made by ``oracle/gen_golden.py`` through the compiled
reference in ``oracle/_ref``) and against the reference's own known-answer
tests (test_cache.cpp:191-196, test_importance.cpp:31-157, test_rng.cpp:14-30,
test_decoder.cpp:246-289).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module.  The product path (``paper_2603_23914_b200``) never does.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# --------------------------------------------------------------------------
# Philox4x32-10 + Box-Muller  (include/kvpack/rng.hpp:15-98)
# --------------------------------------------------------------------------
_M0, _M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
_W0, _W1 = 0x9E3779B9, 0xBB67AE85
_MASK = np.uint64(0xFFFFFFFF)


def philox_round10(key, ctr):
    """rng.hpp:63-78 — vectorised over the last axis of ``ctr`` (shape (4, n))."""
    k0, k1 = int(key[0]) & 0xFFFFFFFF, int(key[1]) & 0xFFFFFFFF
    c = [np.asarray(x, dtype=np.uint64) & _MASK for x in ctr]
    for _ in range(10):
        p0 = _M0 * c[0]
        p2 = _M1 * c[2]
        lo0, hi0 = p0 & _MASK, p0 >> np.uint64(32)
        lo2, hi2 = p2 & _MASK, p2 >> np.uint64(32)
        c = [hi2 ^ c[1] ^ np.uint64(k0), lo2, hi0 ^ c[3] ^ np.uint64(k1), lo0]
        k0 = (k0 + _W0) & 0xFFFFFFFF
        k1 = (k1 + _W1) & 0xFFFFFFFF
    return [x.astype(np.uint32) for x in c]


def philox_u32(seed: int, stream: int, count: int) -> np.ndarray:
    """Stream of next_u32() draws (rng.hpp:25-32): block b uses counter
    {b, 0, stream_lo, stream_hi} (the 128-bit counter increments from 0)."""
    nblk = (count + 3) // 4
    b = np.arange(nblk, dtype=np.uint64)
    ctr = [b & _MASK, b >> np.uint64(32), np.full(nblk, stream & 0xFFFFFFFF, np.uint64),
           np.full(nblk, (stream >> 32) & 0xFFFFFFFF, np.uint64)]
    out = philox_round10((seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF), ctr)
    return np.stack(out, axis=1).reshape(-1)[:count]


def philox_gaussians(seed: int, stream: int, count: int) -> np.ndarray:
    """next_gaussian() x count (rng.hpp:46-59).  Draw i uses Philox block i//2:
    u1 = (a*2^26+b)/2^53 from words 0,1 and u2 from words 2,3 (next_double,
    rng.hpp:39-43); even i -> r*cos(2*pi*u2), odd i -> r*sin(2*pi*u2).  The
    u1 == 0 redraw (probability 2^-53) is not modelled."""
    npair = (count + 1) // 2
    w = philox_u32(seed, stream, npair * 4).reshape(npair, 4).astype(np.uint64)
    u1 = ((w[:, 0] >> np.uint64(5)).astype(np.float64) * 67108864.0 +
          (w[:, 1] >> np.uint64(6)).astype(np.float64)) * (1.0 / 9007199254740992.0)
    u2 = ((w[:, 2] >> np.uint64(5)).astype(np.float64) * 67108864.0 +
          (w[:, 3] >> np.uint64(6)).astype(np.float64)) * (1.0 / 9007199254740992.0)
    r = np.sqrt(-2.0 * np.log(u1))
    ang = 6.283185307179586476925286766559 * u2
    out = np.empty(npair * 2)
    out[0::2] = r * np.cos(ang)
    out[1::2] = r * np.sin(ang)
    return out[:count]


def gaussian_matrix(rows, cols, seed, stream=0):
    """linalg.cpp:175-182 (row-major fill)."""
    return philox_gaussians(seed, stream, rows * cols).reshape(rows, cols)


SVD_STREAM = 0x72737664  # linalg.cpp:77


# --------------------------------------------------------------------------
# Closed forms (cache.cpp:221-229, importance.cpp:119-133)
# --------------------------------------------------------------------------
def compression_ratio(tokens, width, rank):
    if tokens == 0 or width == 0:
        raise ValueError("compression_ratio: token count and width must be positive")
    if rank == 0:
        return 1.0
    return float(tokens) * float(width) / (float(tokens) * float(rank) + float(rank) * float(width))


def flops_partial_decompress(tokens, width, ratios, ranks):
    if not ratios or len(ratios) != len(ranks):
        raise ValueError("flops_partial_decompress: ratios and ranks must align")
    wr = 0.0
    for r, k in zip(ratios, ranks):
        wr += r * float(k)
    flops = int(round_half_away(2.0 * float(tokens) * float(width) * wr))
    red = 0.0 if ranks[0] == 0 else 1.0 - wr / float(ranks[0])
    return flops, red


def round_half_away(x):  # std::llround
    return math.floor(x + 0.5) if x >= 0 else -math.floor(-x + 0.5)


# --------------------------------------------------------------------------
# Importance EMA and grouping (importance.cpp:33-117)
# --------------------------------------------------------------------------
def update_importance(scores, attn, alpha):
    """importance.cpp:33-65.  Rows of attn (T_q x n) must sum to 1 within 1e-4.
    Evaluated in the reference's order: mean = (sum_t a_t) * (1/T_q), then
    decay*s + blend*mean with two separate roundings (no fused multiply-add)."""
    attn = np.atleast_2d(np.asarray(attn, dtype=np.float64))
    s = np.asarray(scores, dtype=np.float64).copy()
    tq = attn.shape[0]
    if attn.shape[1] != s.shape[0]:
        raise ValueError("update_importance: attention width does not match table size")
    if tq == 0:
        return s
    if not (0.0 <= alpha <= 1.0):
        raise ValueError("update_importance: alpha must be in [0, 1]")
    if not np.all(np.isfinite(attn)):
        raise ValueError("update_importance: non-finite attention")
    for t in range(tq):
        rs = 0.0
        for a in attn[t]:
            rs += float(a)
        if abs(rs - 1.0) > 1e-4:
            raise ValueError("update_importance: attention row is not a distribution")
    decay = math.pow(alpha, float(tq))
    blend = 1.0 - decay
    inv_tq = 1.0 / float(tq)
    mean = np.zeros_like(s)
    for t in range(tq):
        mean = mean + attn[t]
    mean = mean * inv_tq
    return decay * s + blend * mean  # numpy evaluates the products separately (no FMA)


def group_sizes(n, ratios):
    """importance.cpp:98-110: floor(r_f*n + 0.5), last group takes the rest."""
    sizes, cursor = [], 0
    for f, r in enumerate(ratios):
        if f + 1 == len(ratios):
            take = n - cursor
        else:
            take = min(int(math.floor(r * float(n) + 0.5)), n - cursor)
        sizes.append(take)
        cursor += take
    return sizes


def assign_groups(scores, ratios, ranks, positions=None):
    """importance.cpp:67-117.  Returns tier_of[i] for each compressed token i
    (masks[f] = sorted indices with tier f).  Order: score descending, ties
    by ascending sequence position."""
    if not ratios or len(ratios) != len(ranks):
        raise ValueError("assign_groups: ratios and ranks must be non-empty and aligned")
    if any(not (r >= 0.0) for r in ratios):
        raise ValueError("assign_groups: ratios must be non-negative")
    tot = 0.0
    for r in ratios:
        tot += r
    if abs(tot - 1.0) > 1e-9:
        raise ValueError("assign_groups: ratios must sum to 1")
    for f in range(1, len(ranks)):
        if ranks[f] > ranks[f - 1]:
            raise ValueError("assign_groups: ranks must be non-increasing")
    s = np.asarray(scores, dtype=np.float64)
    n = s.shape[0]
    pos = np.arange(n) if positions is None else np.asarray(positions, dtype=np.uint64)
    order = np.lexsort((pos, -s))  # primary: -score, secondary: position
    tier = np.zeros(n, dtype=np.uint32)
    cursor = 0
    for f, take in enumerate(group_sizes(n, ratios)):
        tier[order[cursor:cursor + take]] = f
        cursor += take
    return tier


def masks_from_tiers(tier, groups):
    return [np.flatnonzero(tier == f).astype(np.uint32) for f in range(groups)]


def resolved_tier_rank(fraction, stored_rank):
    """decoder.cpp:18-23."""
    if stored_rank == 0:
        return 0
    r = int(math.floor(fraction * float(stored_rank) + 0.5))
    return min(max(r, 1), stored_rank)


# --------------------------------------------------------------------------
# Cache model + retrieval plan (cache.hpp:37-146, decoder.cpp:105-188)
# --------------------------------------------------------------------------
@dataclass
class Store:
    """One BlockStore (cache.hpp:35-60): low-rank factors or dense rows."""
    left: np.ndarray | None = None    # T x R (sigma folded in)
    right: np.ndarray | None = None   # R x W
    rows: np.ndarray | None = None    # T x W (dense)

    @property
    def rank(self):
        return 0 if self.rows is not None else self.left.shape[1]

    def row(self, j, use_rank=0):
        """cache.cpp:63-101 row decompression at a rank prefix (0 = stored)."""
        if self.rows is not None:
            return self.rows[j]
        r = self.rank if use_rank == 0 else min(use_rank, self.rank)
        return self.left[j, :r] @ self.right[:r]


@dataclass
class Block:
    positions: np.ndarray
    keys: Store
    values: Store


@dataclass
class Segment:
    blocks: list = field(default_factory=list)
    tail_k: np.ndarray | None = None
    tail_v: np.ndarray | None = None
    tail_positions: np.ndarray | None = None

    def compressed_positions(self):
        if not self.blocks:
            return np.zeros(0, dtype=np.uint64)
        return np.concatenate([b.positions for b in self.blocks])


@dataclass
class Tiering:
    ratios: list
    key_fractions: list
    value_fractions: list


def resolve_tiering(scores_by_pos: dict, seg: Segment, tiering: Tiering | None):
    """decoder.cpp:105-139 -> (tier_of per compressed row, key_ranks, value_ranks)."""
    pos = seg.compressed_positions()
    if pos.size == 0:
        return None, [], []
    sk, sv = seg.blocks[0].keys.rank, seg.blocks[0].values.rank
    if tiering is None:
        return np.zeros(pos.size, np.uint32), [sk], [sv]
    kr = [resolved_tier_rank(f, sk) for f in tiering.key_fractions]
    vr = [resolved_tier_rank(f, sv) for f in tiering.value_fractions]
    basis = vr if sv > 0 else kr
    scores = np.array([scores_by_pos[int(p)] for p in pos])
    return assign_groups(scores, tiering.ratios, basis, pos), kr, vr


def build_retrieval_plan(segments, scores_by_pos, tiering=None):
    """decoder.cpp:141-188.  Entries: (segment, block, row, rank_k, rank_v,
    position); block = -1 for tail rows.  Order: per segment (visual, textual),
    group-1 rows, lower groups, then tail rows."""
    plan = []
    for s_idx, seg in enumerate(segments):
        tier, kr, vr = resolve_tiering(scores_by_pos, seg, tiering)
        if seg.blocks:
            locate = [(b, r) for b, blk in enumerate(seg.blocks) for r in range(len(blk.positions))]
            for f in range(len(kr)):
                for row in np.flatnonzero(tier == f):
                    b, local = locate[row]
                    blk = seg.blocks[b]
                    plan.append((s_idx, b, local, min(kr[f], blk.keys.rank), min(vr[f], blk.values.rank),
                                 int(blk.positions[local])))
        if seg.tail_positions is not None:
            for r, p in enumerate(seg.tail_positions):
                plan.append((s_idx, -1, r, 0, 0, int(p)))
    return np.array(plan, dtype=np.int64).reshape(-1, 6)


def plan_rows(segments, plan, kind):
    """plan_row (decoder.cpp:27-39) for every entry: the rebuilt K~ or V~."""
    out = []
    for s_idx, b, row, rk, rv, _ in plan:
        seg = segments[s_idx]
        if b < 0:
            out.append((seg.tail_k if kind == 0 else seg.tail_v)[row])
        else:
            st = seg.blocks[b].keys if kind == 0 else seg.blocks[b].values
            out.append(st.row(row, rk if kind == 0 else rv))
    return np.array(out)


def attend_materialized(ktilde, vtilde, positions, queries, qpos, heads, kv_heads, head_dim):
    """decoder.cpp:190-254 in float64: causal visibility by position, logits
    scaled by 1/sqrt(D), max-shifted softmax; returns (context T_q x H*D,
    head_avg T_q x n)."""
    q = np.atleast_2d(np.asarray(queries, dtype=np.float64))
    n = ktilde.shape[0]
    per_kv = heads // kv_heads
    inv_sqrt_d = 1.0 / math.sqrt(float(head_dim))
    ctx = np.zeros((q.shape[0], heads * head_dim))
    ha = np.zeros((q.shape[0], n))
    for i in range(q.shape[0]):
        vis = np.asarray(positions, dtype=np.uint64) <= np.uint64(qpos[i])
        for h in range(heads):
            g = h // per_kv
            kh = ktilde[:, g * head_dim:(g + 1) * head_dim]
            vh = vtilde[:, g * head_dim:(g + 1) * head_dim]
            logit = (kh @ q[i, h * head_dim:(h + 1) * head_dim]) * inv_sqrt_d
            logit = np.where(vis, logit, -np.inf)
            e = np.exp(logit - logit[vis].max())
            z = e.sum()
            ctx[i, h * head_dim:(h + 1) * head_dim] = (e @ vh) / z
            ha[i] += e / z / heads
    return ctx, ha


def attend_lowrank(segments, plan, queries, qpos, heads, kv_heads, head_dim):
    """The same attention evaluated the way the B200 kernels do it — in the
    low-rank space (P = right_k q, S = left_k P, U = p left_v, out = U right_v)
    — used by the tests to show the two formulations agree on the oracle side."""
    return attend_materialized(plan_rows(segments, plan, 0), plan_rows(segments, plan, 1), plan[:, 5],
                               queries, qpos, heads, kv_heads, head_dim)


# --------------------------------------------------------------------------
# Truncated SVD (linalg.cpp:15-114)
# --------------------------------------------------------------------------
def _check_svd(a, rank):
    if a.size == 0:
        raise ValueError("truncated_svd: matrix must be non-empty")
    if rank < 1 or rank > min(a.shape):
        raise ValueError("truncated_svd: rank must be in [1, min(rows, cols)]")
    if not np.all(np.isfinite(a)):
        raise ValueError("truncated_svd: matrix contains non-finite values")


def truncated_svd(a, rank, method="exact", seed=0, oversampling=8, power_iterations=2):
    """linalg.cpp:109-114 -> (left T x R with sigma folded, right R x W orthonormal rows)."""
    a = np.asarray(a, dtype=np.float64)
    _check_svd(a, rank)
    if not np.any(a):  # linalg.cpp:51-59 zero-matrix convention
        right = np.zeros((rank, a.shape[1]))
        right[np.arange(rank), np.arange(rank)] = 1.0
        return np.zeros((a.shape[0], rank)), right
    if method == "exact":  # linalg.cpp:48-63
        u, s, vt = np.linalg.svd(a, full_matrices=False)
        return u[:, :rank] * s[:rank], vt[:rank].copy()
    k = min(rank + oversampling, min(a.shape))  # linalg.cpp:72
    omega = gaussian_matrix(a.shape[1], k, seed, SVD_STREAM)
    q, _ = np.linalg.qr(a @ omega)
    for _ in range(power_iterations):  # linalg.cpp:87-90
        q, _ = np.linalg.qr(a.T @ q)
        q, _ = np.linalg.qr(a @ q)
    b = q.T @ a
    ub, s, vt = np.linalg.svd(b, full_matrices=False)
    return (q @ ub)[:, :rank] * s[:rank], vt[:rank].copy()


# --------------------------------------------------------------------------
# Synthetic workload (harness.cpp:29-32, 82-128, 130-173)
# --------------------------------------------------------------------------
def stream_id(purpose, instance, layer, extra):
    return (purpose << 56) | (instance << 24) | (layer << 8) | extra


def latent_factor_matrix(tokens, kv_heads, head_dim, true_rank, decay, shared, noise, seed, stream):
    """harness.cpp:82-128: one Philox stream consumed in order z (T x r, latent
    i scaled by decay^i), shared loadings (shared x D), per-head loadings
    (kv_heads x (r-shared) x D), then additive noise (T x W)."""
    width = kv_heads * head_dim
    shared = min(shared, true_rank)
    if tokens == 0:
        return np.zeros((0, width))
    n_z = tokens * true_rank
    n_s = shared * head_dim
    n_h = kv_heads * (true_rank - shared) * head_dim
    n_e = tokens * width if noise > 0.0 else 0
    g = philox_gaussians(seed, stream, n_z + n_s + n_h + n_e)
    scale = np.ones(true_rank)
    for i in range(1, true_rank):
        scale[i] = scale[i - 1] * decay
    z = g[:n_z].reshape(tokens, true_rank) * scale
    sh = g[n_z:n_z + n_s].reshape(shared, head_dim)
    hr = g[n_z + n_s:n_z + n_s + n_h].reshape(kv_heads, true_rank - shared, head_dim)
    out = np.zeros((tokens, width))
    for h in range(kv_heads):
        out[:, h * head_dim:(h + 1) * head_dim] = z[:, :shared] @ sh + z[:, shared:] @ hr[h]
    if noise > 0.0:
        out = out + noise * g[n_z + n_s + n_h:].reshape(tokens, width)
    return out
