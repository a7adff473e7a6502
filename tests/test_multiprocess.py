"""World-size-2 checks of the multi-GPU host logic on CPU (gloo): instance
sharding covers the stream exactly once, and the result gather reassembles
per-rank outputs in rank order."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1711_11407_b200.shard import gather_results, instance_range


def test_instance_range_partitions():
    for total in (0, 1, 7, 4096):
        for world in (1, 2, 3, 8):
            spans = [instance_range(r, world, total=total) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    assert instance_range(3, 8, per_rank=4096) == (3 * 4096, 4 * 4096)
    with pytest.raises(ValueError):
        instance_range(2, 2, total=4)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        b0, b1 = instance_range(rank, world, per_rank=3)
        n = b1 - b0
        outs = {
            "count": torch.arange(b0, b1, dtype=torch.int32),
            "iterations": torch.full((n,), rank + 1, dtype=torch.int32),
            "samples_used": torch.full((n,), 768 * (rank + 1), dtype=torch.int64),
            "terminated_by": torch.zeros(n, dtype=torch.int32),
            "freqs": torch.full((n, 4, 2), rank, dtype=torch.int32),
            "amps": torch.full((n, 4), complex(rank, -rank), dtype=torch.complex128),
        }
        got = gather_results(outs)
        if rank == 0:
            q.put((got["count"].tolist(), got["iterations"].tolist(),
                   got["amps"][:, 0].tolist(), tuple(got["freqs"].shape)))
        else:
            q.put(got)
    finally:
        dist.destroy_process_group()


def test_gather_results_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res = [r for r in res if r is not None]
    assert len(res) == 1
    counts, iters, amps, fshape = res[0]
    assert counts == list(range(6))
    assert iters == [1, 1, 1, 2, 2, 2]
    assert amps == [0j, 0j, 0j, (1 - 1j), (1 - 1j), (1 - 1j)]
    assert fshape == (6, 4, 2)
