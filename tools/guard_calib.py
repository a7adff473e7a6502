#!/usr/bin/env python
"""Calibrate the guard band of precision="fp32-guarded" (csrc/fpssft_guard.cuh).

Needs the calibration build (every candidate bin is re-evaluated exactly and
the float32 error of its D+1 values is recorded in units of the kappa = 1
bound):
    nvcc ... -DFPSSFT_GUARD_CALIB=1 -o build/libfpssft_calib.so csrc/fpssft.cu
    FPSSFT_LIB=build/libfpssft_calib.so python tools/guard_calib.py
Prints, per config, the largest observed error / bound and the bins measured:
the shipped kappa (FPSSFT_GUARD_KF / _KP) must sit well above it."""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="5,3")
    ap.add_argument("--count", type=int, default=256)
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_1711_11407_b200 as P
    from paper_1711_11407_b200 import _native as N
    from paper_1711_11407_b200 import workloads as W

    lib = N.lib()
    lib.fpssft_guard_calib.argtypes = [C.POINTER(C.c_float), C.POINTER(C.c_ulonglong)]
    mx, cnt = C.c_float(), C.c_ulonglong()
    lib.fpssft_guard_calib(C.byref(mx), C.byref(cnt))  # reset
    for c in [int(x) for x in args.configs.split(",")]:
        w = W.CONFIGS[c]
        spectra = W.make_spectra(w, args.count, 0)
        cubes = W.synthesize_batch_torch(w.dims, spectra, "cuda", w.noise_var,
                                         noise_seed=w.seed * 1000003)
        for mode in ("cta", "warp") if c == 3 else ("auto",):
            cfg = P.FpsSftConfig(seed=c, **P.PROFILES[w.profile])
            res = P.fps_sft_batch(cubes, cfg, k_cap=1024, precision="fp32-guarded", mode=mode)
            torch.cuda.synchronize()
            lib.fpssft_guard_calib(C.byref(mx), C.byref(cnt))
            print(json.dumps({"lib": os.path.basename(N.LIB_PATH), "config": c, "mode": mode, "instances": args.count,
                              "bins_measured": cnt.value, "max_error_over_unit_bound": mx.value,
                              "kappa_f": float(os.environ.get("KF", 6.0)), "mean_iterations":
                              float(res.iterations.float().mean())}), flush=True)


if __name__ == "__main__":
    main()
