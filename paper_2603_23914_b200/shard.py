"""Instance sharding across GPUs (one process per GPU) and the once-per-run
gather of results.

The reference parallelises one way only: a thread pool over batch instances
with an instance-ordered merge of their reports (harness.cpp:364-441,
`run_experiment`: atomic work counter, per-instance results written to slot
`i`, merged in instance order).  Instances share nothing, so here they are
split contiguously across ranks and each rank decodes its own
slice with no collective on the per-step path.  The only collective on the
data path is one gather of per-instance outputs and step records to rank 0 at
the end of the run (NCCL on a GPU box, gloo in the CPU tests), merged in global
instance order exactly like the reference's ordered merge.
"""
from __future__ import annotations


def instance_range(global_batch: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [lo, hi) slice of the global batch owned by `rank`.

    Sizes differ by at most one when the batch does not divide (the first
    `global_batch % world` ranks take one more), so every instance is owned by
    exactly one rank and rank order is instance order."""
    if global_batch < 1 or world < 1 or not 0 <= rank < world:
        raise ValueError("instance_range: need global_batch >= 1, world >= 1, 0 <= rank < world")
    if global_batch < world:
        raise ValueError(f"instance_range: {global_batch} instances cannot be split over {world} ranks")
    base, extra = divmod(global_batch, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def gather_instances(local, world: int, global_batch: int):
    """Gather every rank's per-instance rows (a torch tensor [n_local, ...]) to
    rank 0 and return them merged in global instance order ([global_batch, ...]);
    other ranks return None.  One collective: an all_gather of fixed-size,
    padded blocks (NCCL needs equal sizes), trimmed by the known slice sizes."""
    import torch
    import torch.distributed as dist

    if world == 1:
        return local
    rank = dist.get_rank()
    sizes = [instance_range(global_batch, world, r)[1] - instance_range(global_batch, world, r)[0]
             for r in range(world)]
    cap = max(sizes)
    pad = torch.zeros((cap,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    blocks = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(blocks, pad)
    if rank != 0:
        return None
    return torch.cat([b[:n] for b, n in zip(blocks, sizes)], dim=0)
