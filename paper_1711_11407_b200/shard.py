"""Multi-GPU plumbing: instances are independent, so each rank (one process
per GPU) owns a contiguous slice of the instance stream and runs it with no
data-path communication.  The only collective on the data is the optional
final gather of the padded per-instance results to rank 0 (SURVEY.md section
8(e)), issued through ``torch.distributed`` (NCCL over NVLink on B200; gloo
on CPU in the tests).  This replaces the reference's instance-parallel
``ProcessPoolExecutor`` (``pkg/src/fps_sft/oracle.py:275-277``): trials
farmed to workers become batch slices farmed to GPUs.

``launch`` starts the ranks: under ``torchrun`` (``WORLD_SIZE`` set) the
calling process is one rank; otherwise it spawns ``n`` processes itself,
each with ``RANK``/``LOCAL_RANK``/``WORLD_SIZE``/``MASTER_*`` set the way
``torchrun`` would, so ``bench.py --gpus N`` is a real N-rank run either way.
"""

from __future__ import annotations

import os
import socket


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


def env_rank() -> tuple[int, int, int]:
    """(rank, local_rank, world) from the torchrun-style environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spawned(local: int, n: int, port: int, fn, args) -> None:
    os.environ.update(RANK=str(local), LOCAL_RANK=str(local), WORLD_SIZE=str(n),
                      LOCAL_WORLD_SIZE=str(n), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    fn(*args)


def launch(n: int, fn, *args) -> None:
    """Run ``fn(*args)`` on ``n`` ranks.  Under torchrun (``WORLD_SIZE`` in
    the environment) this process is already one rank: call ``fn`` once and
    check the world matches ``n``.  Otherwise ``n == 1`` calls ``fn`` here
    and ``n > 1`` spawns ``n`` processes (torch.multiprocessing, ``spawn``
    start method) and waits for all of them; a failing rank raises."""
    if "WORLD_SIZE" in os.environ:
        world = int(os.environ["WORLD_SIZE"])
        if world != n:
            raise ValueError(f"--gpus {n} but the launcher started {world} ranks")
        fn(*args)
        return
    if n == 1:
        fn(*args)
        return
    import torch.multiprocessing as mp

    mp.spawn(_spawned, args=(n, _free_port(), fn, args), nprocs=n, join=True)


RESULT_FIELDS = ("count", "iterations", "samples_used", "terminated_by", "freqs", "amps")


def result_bytes(outputs: dict) -> int:
    return sum(outputs[k].numel() * outputs[k].element_size() for k in RESULT_FIELDS)


def gather_results(outputs: dict, dst: int = 0, group=None) -> dict | None:
    """Gather each rank's padded per-instance result tensors (``BatchResult``
    / ``allocate_outputs`` fields, equal batch per rank) to rank ``dst``
    (``torch.distributed.gather``: only ``dst`` receives).  Returns the
    rank-ordered concatenation on ``dst`` and None elsewhere."""
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
        parts = [torch.empty_like(t) for _ in range(world)] if rank == dst else None
        dist.gather(t, parts, dst=dst, group=group)
        if rank == dst:
            cat = torch.cat(parts, dim=0)
            if outputs[name].is_complex():
                cat = torch.view_as_complex(cat)
            out[name] = cat
    return out if rank == dst else None


def max_over_ranks(value: float, device=None, group=None) -> float:
    """The largest ``value`` over all ranks (elapsed times: a multi-GPU step
    takes as long as its slowest rank)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
