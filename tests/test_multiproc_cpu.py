"""The N > 1 plumbing of bench.py on CPU: world size 2 over gloo (127.0.0.1).
Instances are sharded across ranks with no data-path collective (SURVEY.md
§8e); the only collectives are the barrier and the max over ranks of the
device-timed region, and `value` aggregates every rank's tokens."""
import os
import socket
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port), CUDA_VISIBLE_DEVICES="")
    sys.path.insert(0, str(ROOT))
    import bench
    import torch.distributed as dist
    w, r, _ = bench.dist_setup()
    bench.barrier(w)
    ms = bench.max_over_ranks(10.0 + r, w)  # rank 1 is the slower one
    value = bench.aggregate_throughput(w, 16, 20, ms)
    q.put((r, w, dist.get_backend(), ms, value))
    dist.destroy_process_group()


def test_two_rank_max_over_ranks_and_weak_scaling():
    mp = pytest.importorskip("torch.multiprocessing")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [o[0] for o in out] == [0, 1]
    for r, w, backend, ms, value in out:
        assert (w, backend) == (2, "gloo")
        assert ms == 11.0  # max over ranks, identical on every rank
        assert value == pytest.approx(2 * 16 * 20 / 11e-3)


def _gather_worker(rank, world, port, gb, q):
    os.environ.update(RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port), CUDA_VISIBLE_DEVICES="")
    sys.path.insert(0, str(ROOT))
    import bench
    import torch
    import torch.distributed as dist
    from paper_2603_23914_b200.shard import gather_instances
    w, r, _ = bench.dist_setup()
    cfg = dict(bench.CONFIGS["c3"])
    total, lo, hi, scaling = bench.shard_plan(cfg, w, r, gb)
    # stand-in for the per-instance decode output: a pure function of the global instance index
    local = torch.stack([torch.arange(8, dtype=torch.float64) * (i + 1) + i for i in range(lo, hi)])
    out = gather_instances(local, w, total)
    q.put((r, lo, hi, scaling, None if out is None else out.numpy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("gb", [64, 7])
def test_two_rank_instance_sharding_and_ordered_gather(gb):
    """C3-style strong scaling: the global batch is split contiguously (64 -> 32 + 32;
    7 -> 4 + 3) and the once-per-run gather returns every instance's output in global
    instance order on rank 0 — identical to what one rank computing all instances holds."""
    import numpy as np
    mp = pytest.importorskip("torch.multiprocessing")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, 2, port, gb, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted((q.get(timeout=120) for _ in procs), key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, lo0, hi0, sc0, g0), (r1, lo1, hi1, sc1, g1) = out
    assert (lo0, hi0, lo1, hi1) == (0, (gb + 1) // 2, (gb + 1) // 2, gb)
    assert sc0 == sc1 == "strong"
    assert g1 is None
    single = np.stack([np.arange(8, dtype=np.float64) * (i + 1) + i for i in range(gb)])
    assert np.array_equal(g0, single)


def test_instance_range_partitions_the_batch():
    from paper_2603_23914_b200.shard import instance_range
    for gb in (1, 2, 7, 16, 64, 65):
        for world in (1, 2, 4, 8):
            if gb < world:
                with pytest.raises(ValueError):
                    instance_range(gb, world, 0)
                continue
            spans = [instance_range(gb, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == gb
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [h - l for l, h in spans]
            assert max(sizes) - min(sizes) <= 1
    assert instance_range(64, 8, 3) == (24, 32)  # C3: 8 instances per GPU


def test_clock_sampler_window_and_reasons():
    # bench.ClockSampler keeps the samples that bracket the timed region and
    # reports the median SM clock and the throttle reasons seen there.
    import time

    import bench

    s = bench.ClockSampler(0)
    now = time.monotonic()
    s.samples = [(1000.0, 1965.0, 0x0, now - 1.0), (1900.0, 1965.0, 0x0, now - 0.05),
                 (1965.0, 1965.0, 0x4, now + 0.05), (1950.0, 1965.0, 0x0, now + 0.15)]
    s.t_begin = now
    out = s.stop()
    assert out["sm_mhz"] == 1950.0 and out["sm_max_mhz"] == 1965.0
    assert out["reasons"] == ["sw_power_cap"]
