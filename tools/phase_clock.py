#!/usr/bin/env python
"""Per-phase warp time of the warp kernel (FPSSFT_PHASE_CLOCK=1 builds, lib
via FPSSFT_LIB): cycles summed over every warp's lane 0, as shares.
usage: FPSSFT_LIB=build/ab/clock.so tools/phase_clock.py --config 2"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
NAMES = ["gather (group: issue + barrier)", "gather store + barrier", "FFT", "projection (3)",
         "classify (4)", "decode + merge (5)", "amp_sum + termination", "output sort",
         "kernel start (roots; warp kernel: + non-group gathers)",
         "team guarded: flag re-evaluation", "team: exscan + merge", "-"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--layout", default="interleaved")
    ap.add_argument("--precision", default="auto")
    args = ap.parse_args()
    import torch

    import bench
    import paper_1711_11407_b200 as P
    from paper_1711_11407_b200 import _native as N
    from paper_1711_11407_b200 import workloads as W

    w = W.CONFIGS[args.config]
    dev = torch.device("cuda:0")
    spectra = W.make_spectra(w, w.batch, 0)
    cubes = W.synthesize_batch_torch(w.dims, spectra, dev, w.noise_var,
                                     noise_seed=w.seed * 1000003)
    group = 8 if args.layout == "interleaved" else 1
    run_cubes = P.interleave(cubes, group) if group > 1 else cubes
    cfg = bench._cfg(w, args.config)
    r = P.BatchRunner(P.CubeShape(w.dims), cfg, w.batch, k_cap=bench.K_CAP[args.config],
                      precision=args.precision, device=dev, group=group)
    lib = N.lib()
    f = lib.fpssft_debug_phase_cycles
    buf = (ctypes.c_ulonglong * 16)()
    for _ in range(3):
        r.run(run_cubes)
    torch.cuda.synchronize()
    f(buf, 1)
    r.run(run_cubes)
    torch.cuda.synchronize()
    f(buf, 1)
    tot = sum(buf[:12])
    print(f"config {args.config} {args.layout}: {tot / 1e9:.3f} G warp-cycles "
          f"({tot / w.batch / 1e3:.1f} k per instance)")
    for n, v in zip(NAMES, buf[:12]):
        print(f"  {n:30s} {100 * v / tot:5.1f} %  {v / w.batch:9.0f} cycles/instance")


if __name__ == "__main__":
    main()
