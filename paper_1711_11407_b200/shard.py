"""Multi-GPU plumbing: instances are independent, so each rank (one process
per GPU) owns a contiguous slice of the instance stream and runs it with no
data-path communication.  The only collective is the optional final gather
of the padded per-instance results to rank 0,
issued through ``torch.distributed`` (NCCL over NVLink on B200; gloo on CPU
in the tests)."""

from __future__ import annotations


def instance_range(rank: int, world: int, total: int | None = None,
                   per_rank: int | None = None) -> tuple[int, int]:
    """[start, stop) of this rank's instances.  ``per_rank`` (weak scaling):
    every rank gets that many consecutive instances.  ``total`` (strong
    scaling): a near-even contiguous split of ``total``."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    if per_rank is not None:
        return rank * per_rank, (rank + 1) * per_rank
    if total is None:
        raise ValueError("give total or per_rank")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


RESULT_FIELDS = ("count", "iterations", "samples_used", "terminated_by", "freqs", "amps")


def gather_results(outputs: dict, dst: int = 0, group=None) -> dict | None:
    """Gather equal-size per-rank result tensors (``BatchResult`` fields) to
    ``dst`` with ``all_gather_into_tensor`` semantics; returns the
    concatenated dict on ``dst`` and None elsewhere."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    out = {}
    for name in RESULT_FIELDS:
        t = outputs[name]
        if t.is_complex():
            t = torch.view_as_real(t)
        t = t.contiguous()
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t, group=group)
        cat = torch.cat(parts, dim=0)
        if outputs[name].is_complex():
            cat = torch.view_as_complex(cat)
        out[name] = cat
    return out if rank == dst else None
