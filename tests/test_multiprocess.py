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


# ---- the bench's N-rank launcher (shard.launch) end to end on CPU ranks
def _bench_like_rank(out_path, total):
    """One rank of a strong-scaled job: its contiguous slice of ``total``
    tiny instances recovered (by the CPU oracle, standing in for the device
    kernel), padded results gathered to rank 0, the time reduced as a max."""
    import numpy as np

    from oracle import fps_oracle as O
    from paper_1711_11407_b200 import shard
    from paper_1711_11407_b200 import workloads as W

    rank, local, world = shard.env_rank()
    dist.init_process_group("gloo")
    try:
        b0, b1 = shard.instance_range(rank, world, total=total)
        outs = _oracle_outputs(W, O, np, b0, b1)
        got = shard.gather_results(outs)
        t = shard.max_over_ranks(float(rank + 1))
        if rank == 0:
            torch.save({"world": world, "span": (b0, b1), "t": t,
                        **{k: v for k, v in got.items()}}, out_path)
    finally:
        dist.destroy_process_group()


def _oracle_outputs(W, O, np, b0, b1, k_cap=16):
    dims = (16, 12)
    w = W.Workload("t", dims, b1 - b0, 6, "uniform", "unit", 0.0, "P32", 77)
    n = b1 - b0
    outs = {"count": torch.zeros(n, dtype=torch.int32),
            "iterations": torch.zeros(n, dtype=torch.int32),
            "samples_used": torch.zeros(n, dtype=torch.int64),
            "terminated_by": torch.zeros(n, dtype=torch.int32),
            "freqs": torch.zeros((n, k_cap, 2), dtype=torch.int32),
            "amps": torch.zeros((n, k_cap), dtype=torch.complex128)}
    for j, r in enumerate(W.instance_rngs(77, n, b0)):
        _, _, cube = W.make_instance(w, r)
        rep = O.recover(cube, dims, O.P32, seed=5)
        c = len(rep.amps)
        outs["count"][j] = c
        outs["iterations"][j] = rep.iterations_run
        outs["samples_used"][j] = rep.samples_used
        outs["freqs"][j, :c] = torch.as_tensor(rep.freqs.astype(np.int32))
        outs["amps"][j, :c] = torch.as_tensor(rep.amps)
    return outs


def test_launch_spawns_world2_and_gathers(tmp_path):
    """``shard.launch(2, ...)`` without torchrun spawns two ranks with the
    torchrun environment; their disjoint slices gather on rank 0 into the
    single-rank result, and the job time is the max over ranks."""
    import numpy as np

    from oracle import fps_oracle as O
    from paper_1711_11407_b200 import shard
    from paper_1711_11407_b200 import workloads as W

    out = str(tmp_path / "r0.pt")
    env = {k: os.environ.pop(k) for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK") if k in os.environ}
    try:
        shard.launch(2, _bench_like_rank, out, 6)
    finally:
        os.environ.update(env)
    got = torch.load(out)
    assert got["world"] == 2 and tuple(got["span"]) == (0, 3) and got["t"] == 2.0
    want = _oracle_outputs(W, O, np, 0, 6)
    for k, v in want.items():
        assert torch.equal(got[k], v), k


def test_launch_under_torchrun_env_checks_world(monkeypatch):
    from paper_1711_11407_b200 import shard

    monkeypatch.setenv("WORLD_SIZE", "4")
    with pytest.raises(ValueError):
        shard.launch(2, lambda: None)
    seen = []
    monkeypatch.setenv("WORLD_SIZE", "2")
    shard.launch(2, lambda x: seen.append(x), 7)
    assert seen == [7]
