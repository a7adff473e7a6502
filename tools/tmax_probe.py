#!/usr/bin/env python
"""Launch time of the config-2 group kernel with the loop cut at t_max = T
(what a first phase that stops after T iterations costs), and of a small
batch-major launch (a straggler phase).  Timing only; outputs not checked."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timeit(fn, n=20):
    import torch

    flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for i in range(n):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[n // 2]


def main():
    import dataclasses

    import torch

    import bench
    import paper_1711_11407_b200 as P
    from paper_1711_11407_b200 import workloads as W

    w = W.CONFIGS[2]
    dev = torch.device("cuda:0")
    spectra = W.make_spectra(w, w.batch, 0)
    cubes = W.synthesize_batch_torch(w.dims, spectra, dev, 0.0, noise_seed=0)
    il = P.interleave(cubes, 8)
    cfg = bench._cfg(w, 2)
    for T in (0, 2, 3, 4):
        c = cfg if T == 0 else dataclasses.replace(cfg, max_iterations=T)
        r = P.BatchRunner(P.CubeShape(w.dims), c, w.batch, k_cap=128, device=dev, group=8)
        print(f"group kernel, t_max {T or 'default'}: {timeit(lambda: r.run(il)):.4f} ms", flush=True)
    for nb in (256, 512):
        c = dataclasses.replace(cfg, max_iterations=2)
        r = P.BatchRunner(P.CubeShape(w.dims), c, nb, k_cap=128, device=dev)
        sub = cubes[:nb].contiguous()
        print(f"batch-major {nb} instances, t_max 2: {timeit(lambda: r.run(sub)):.4f} ms", flush=True)


if __name__ == "__main__":
    main()
