#!/usr/bin/env python
"""A/B of the host-buffer paths (config N, one GPU): HostBatchRunner in
copy / zero_copy / split(f) / auto mode against the device-resident run.
Prints ms per batch for each and whether every output (and, for config 5,
every re-synthesised image) equals the device-resident results bit for bit.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--fractions", default="0.3,0.5,0.65,0.8")
    args = ap.parse_args()
    import torch

    import paper_1711_11407_b200 as P
    from paper_1711_11407_b200 import ops
    from paper_1711_11407_b200 import workloads as W
    from paper_1711_11407_b200.hostpath import HostBatchRunner

    K_CAP = {1: 64, 2: 128, 3: 512, 4: 2048, 5: 1024}
    w = W.CONFIGS[args.config]
    B = args.batch or w.batch
    dev = torch.device("cuda:0")
    shape = P.CubeShape(w.dims)
    spectra = W.make_spectra(w, B, 0)
    cubes = W.synthesize_batch_torch(w.dims, spectra, dev, w.noise_var, noise_seed=w.seed)
    cfg = P.FpsSftConfig(seed=args.config, **P.PROFILES[w.profile])
    kc = K_CAP[args.config]
    runner = P.BatchRunner(shape, cfg, B, k_cap=kc, device=dev)
    host = torch.empty(cubes.shape, dtype=cubes.dtype, pin_memory=True)
    host.copy_(cubes)
    synth = args.config == 5
    images = torch.empty(cubes.shape, dtype=cubes.dtype, pin_memory=True) if synth else None
    r = runner.run(cubes)
    ref = {k: v.cpu() for k, v in runner.out.items() if v is not None}
    ref_img = None
    if synth:
        ref_img = ops.synthesize(r).cpu()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.reps):
        r = runner.run(cubes)
        if synth:
            ops.synthesize(r)
    b.record()
    b.synchronize()
    out = {"config": args.config, "batch": B, "dev_ms": a.elapsed_time(b) / args.reps,
           "mean_samples": float(ref["samples_used"].double().mean())}
    modes = [("copy", None), ("zero_copy", None)] + \
        [("split", float(f)) for f in args.fractions.split(",")] + [("auto", None)]
    for mode, f in modes:
        hr = HostBatchRunner(shape, cfg, B, k_cap=kc, device=dev, mode=mode,
                             zero_copy_fraction=f)
        hr.run(host, images)  # warm (auto: learns the sample count)
        ts = []
        for _ in range(args.reps):
            t0 = time.perf_counter()
            o = hr.run(host, images)
            ts.append((time.perf_counter() - t0) * 1e3)
        eq = all(torch.equal(ref[k], o[k]) for k in ref)
        if synth:
            eq = eq and bool(torch.equal(ref_img, images))
        key = mode if f is None else f"split{f}"
        out[key] = {"ms": min(ts), "mean_ms": sum(ts) / len(ts), "equal": eq,
                    "zero_copy_instances": hr.split_count()}
        del hr
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
