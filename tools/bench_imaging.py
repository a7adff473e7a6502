#!/usr/bin/env python
"""Imaging duality path timing: the paper's 512 x 576
phantom at its three sparsity levels, GPU (reconstruct_sparse_image:
device DFT + fps_sft_large, float64) vs the CPU oracle port of the same loop
(numpy float64, one core) on this host.  One JSON line per level.

usage: PYTHONPATH=. python tools/bench_imaging.py [--reps 3]"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from oracle import fps_oracle as O
    from paper_1711_11407_b200 import FpsSftConfig
    from paper_1711_11407_b200 import imaging as I
    from paper_1711_11407_b200.driver import default_max_iterations

    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--loop", default="device", choices=["device", "host"])
    args = ap.parse_args()
    ph = I.synthetic_phantom((512, 576), 1)
    for level, target in enumerate((0.0285, 0.0448, 0.0661)):
        sparse = I.sparsify(ph, I.threshold_for_fraction(ph, target))
        cfg = FpsSftConfig(stall_limit=10, seed=800 + level)
        I.reconstruct_sparse_image(sparse, cfg, loop=args.loop)  # warm-up
        ts = []
        for _ in range(args.reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            recon, rep = I.reconstruct_sparse_image(sparse, cfg, loop=args.loop)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        err = float(np.abs(recon.pixels - sparse.pixels).max())
        # CPU: the oracle port of the same loop on the same (numpy) frequency cube
        n = sparse.pixels.size
        k = int(np.count_nonzero(sparse.pixels))
        t_max = max(default_max_iterations(I.CubeShape((512, 576))), -(-4 * k // 4608) + 20)
        prof = O.Profile(amp_prune_tol=cfg.amp_prune_tol / n, energy_floor_abs=cfg.energy_floor_abs / n, stall_limit=10,
                         max_iterations=t_max)
        t0 = time.perf_counter()
        xhat = np.fft.fftn(sparse.pixels.astype(np.complex128)) / n
        ref = O.recover(xhat, (512, 576), prof, seed=800 + level)
        cpu = time.perf_counter() - t0
        print(json.dumps(dict(loop=args.loop, level=level, k=k, iterations=rep.iterations_run,
                              terminated_by=rep.terminated_by,
                              percent_samples=rep.percent_samples(), max_pixel_error=err,
                              gpu_s=min(ts), gpu_ms_per_iteration=1e3 * min(ts) / rep.iterations_run,
                              cpu_oracle_s=cpu, cpu_iterations=ref.iterations_run,
                              speedup=cpu / min(ts))), flush=True)


if __name__ == "__main__":
    main()
