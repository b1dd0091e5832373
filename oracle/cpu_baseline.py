"""ORACLE / TEST INFRASTRUCTURE ONLY — the CPU reference arm of bench.py.

Times the reference's own decode step (decoder.cpp:555-617 via the compiled
reference in oracle/_ref, engine precision f32 like the reference harness
default) on a bounded sample of the benchmark workload: `threads` independent
(instance, layer) caches of the exact benchmark geometry, each compacted by the
reference's own compress_now (randomized SVD), then one decode_step each, run
in parallel on the host cores exactly like the reference harness parallelises
over instances (harness.cpp:372-398).  Decode tokens/s for the whole job is
extrapolated linearly: one step of all B*L (instance, layer) pairs on
`threads` cores takes B*L/threads * t_pair.
"""
from __future__ import annotations

import os
import threading
import time

import numpy as np

from . import ref
from .cases import decode_ini


def _low_rank_kv(rng, tokens, width, rank):
    """Fast synthetic prefill with a decaying spectrum (values do not change
    the reference's cost, which is data-independent)."""
    u = rng.standard_normal((tokens, 2 * rank)).astype(np.float32)
    v = rng.standard_normal((2 * rank, width)).astype(np.float32) / np.sqrt(width)
    u *= (0.98 ** np.arange(2 * rank, dtype=np.float32))
    return u @ v + 1e-2 * rng.standard_normal((tokens, width)).astype(np.float32)


class ReferenceSample:
    def __init__(self, geom, visual_tokens, textual_tokens, rank_k, rank_v, threads, seed=0, tiering=None):
        H, Hkv, D = geom
        self.geom = geom
        self.threads = threads
        W, HD = Hkv * D, H * D
        self.ini = decode_ini(ranks=(rank_k, rank_v, 0, 0), tiering=tiering, period=512, svd="randomized")
        rng = np.random.default_rng(seed)
        s = 1.0 / np.sqrt(HD)
        self.weights = [rng.standard_normal(sh).astype(np.float32) * s for sh in ((HD, HD), (HD, W), (HD, W), (HD, HD))]
        self.caches = []
        kv = [(_low_rank_kv(rng, visual_tokens, W, rank_k), _low_rank_kv(rng, visual_tokens, W, rank_v),
               rng.standard_normal((textual_tokens, W)).astype(np.float32),
               rng.standard_normal((textual_tokens, W)).astype(np.float32)) for _ in range(threads)]

        def build(i):
            c = ref.RefCache(H, Hkv, D, dtype="f32")
            c.append(0, kv[i][0], kv[i][1])
            if textual_tokens:
                c.append(1, kv[i][2], kv[i][3])
            c.compress_now(self.ini)  # reference compaction (not timed)
            self.caches[i] = c

        self.caches = [None] * threads
        ts = [threading.Thread(target=build, args=(i,)) for i in range(threads)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        self.x = rng.standard_normal((threads, 1, HD)).astype(np.float32)

    def step(self) -> float:
        """One reference decode_step on every sampled cache in parallel; wall seconds."""
        err = []

        def run(i):
            try:
                self.caches[i].decode_step(self.x[i], *self.weights, decode_ini=self.ini)
            except Exception as e:  # surfaced below
                err.append(e)

        ts = [threading.Thread(target=run, args=(i,)) for i in range(self.threads)]
        t0 = time.perf_counter()
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        dt = time.perf_counter() - t0
        if err:
            raise err[0]
        return dt


def tokens_per_second(pair_seconds, batch, layers, threads):
    """Whole-job decode tokens/s: B tokens per step, a step = B*L pairs over `threads` cores."""
    step_s = pair_seconds * batch * layers / threads
    return batch / step_s


def host_threads() -> int:
    return max(1, min(len(os.sched_getaffinity(0)), 64))
