#!/usr/bin/env python
"""Launch the re-synthesis kernel alone on B frames of a config-5-like
spectrum (K entries per frame, uniform support, Rayleigh magnitudes), for
ncu captures and A/B timing: prints ms per launch (CUDA events, warm)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=2048)
    ap.add_argument("--k", type=int, default=500)
    ap.add_argument("--k-cap", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_1711_11407_b200 as P
    from paper_1711_11407_b200 import ops

    rng = np.random.default_rng(5)
    B, K, KC = args.frames, args.k, args.k_cap
    f = np.zeros((B, KC, 2), np.int32)
    a = np.zeros((B, KC), np.complex128)
    for b in range(B):
        lin = rng.choice(512 * 512, K, replace=False)
        f[b, :K, 0], f[b, :K, 1] = lin // 512, lin % 512
        a[b, :K] = rng.rayleigh(1.0, K) * np.exp(2j * np.pi * rng.random(K))
    dev = torch.device("cuda:0")
    ft, at = torch.as_tensor(f, device=dev), torch.as_tensor(a, device=dev)
    ct = torch.full((B,), K, dtype=torch.int32, device=dev)
    out = torch.empty((B, 512, 512), dtype=torch.complex64, device=dev)
    shape = P.CubeShape((512, 512))
    for _ in range(2):
        ops.synthesize(ft, at, ct, shape=shape, out=out)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(args.reps):
        ops.synthesize(ft, at, ct, shape=shape, out=out)
    e.record()
    e.synchronize()
    ms = s.elapsed_time(e) / args.reps
    print(f"synthesize {B} frames: {ms:.3f} ms  {B * 512 * 512 * 8 / ms / 1e6:.0f} GB/s written")


if __name__ == "__main__":
    main()
