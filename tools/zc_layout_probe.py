#!/usr/bin/env python
"""Zero-copy recovery straight from pinned host memory, batch-major vs
interleaved host layouts (config N): ms per batch and bit-equality with the
device-resident batch-major run."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--groups", default="1,8,16,32")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch

    import paper_1711_11407_b200 as P
    from paper_1711_11407_b200 import workloads as W

    K_CAP = {1: 64, 2: 128, 3: 512, 4: 2048, 5: 1024}
    w = W.CONFIGS[args.config]
    B = args.batch or w.batch
    dev = torch.device("cuda:0")
    cubes = W.synthesize_batch_torch(w.dims, W.make_spectra(w, B, 0), dev, w.noise_var,
                                     noise_seed=w.seed)
    cfg = P.FpsSftConfig(seed=args.config, **P.PROFILES[w.profile])
    shape = P.CubeShape(w.dims)
    ref = P.BatchRunner(shape, cfg, B, k_cap=K_CAP[args.config], device=dev)
    ref.run(cubes)
    want = {k: v.cpu() for k, v in ref.out.items() if v is not None}
    out = {"config": args.config, "batch": B}
    for G in [int(g) for g in args.groups.split(",")]:
        src = P.interleave(cubes, G) if G > 1 else cubes
        host = torch.empty(src.shape, dtype=src.dtype, pin_memory=True)
        host.copy_(src)
        del src
        r = P.BatchRunner(shape, cfg, B, k_cap=K_CAP[args.config], device=dev, group=G)
        r.run(host)
        torch.cuda.synchronize()
        ts = []
        for _ in range(args.reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            r.run(host)
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        eq = all(torch.equal(want[k], r.out[k].cpu()) for k in want)
        out[f"G{G}"] = {"ms": min(ts), "equal": eq}
        del host
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
