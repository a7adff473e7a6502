#!/usr/bin/env python
"""Why guarded float32 decisions get flagged (FPSSFT_GUARD_CALIB=2 builds via
FPSSFT_LIB): per config, flags per instance by reason, decodes and certain
bin-map rejections, and the exact re-evaluations (bins) per instance."""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
NAMES = ["magnitude", "phase_uncertain", "rint_either_way", "verify_band", "round_band",
         "decodes", "binmap_rejects"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="3,5")
    ap.add_argument("--count", type=int, default=256)
    args = ap.parse_args()
    import torch

    import bench
    import paper_1711_11407_b200 as P
    from paper_1711_11407_b200 import _native as N
    from paper_1711_11407_b200 import workloads as W

    lib = N.lib()
    buf = (C.c_ulonglong * 8)()
    mx, cnt = C.c_float(), C.c_ulonglong()
    for c in [int(x) for x in args.configs.split(",")]:
        w = W.CONFIGS[c]
        spectra = W.make_spectra(w, args.count, 0)
        cubes = W.synthesize_batch_torch(w.dims, spectra, "cuda", w.noise_var,
                                         noise_seed=w.seed * 1000003)
        lib.fpssft_guard_reasons(buf)
        lib.fpssft_guard_calib(C.byref(mx), C.byref(cnt))
        cfg = P.FpsSftConfig(seed=c, **P.PROFILES[w.profile])
        res = P.fps_sft_batch(cubes, cfg, k_cap=bench.K_CAP[c], precision="fp32-guarded")
        torch.cuda.synchronize()
        lib.fpssft_guard_reasons(buf)
        lib.fpssft_guard_calib(C.byref(mx), C.byref(cnt))
        it = float(res.iterations.float().mean())
        print(json.dumps({"config": c, "instances": args.count, "mean_iterations": it,
                          "per_instance": {n: buf[i] / args.count for i, n in enumerate(NAMES)},
                          "exact_reevaluations_per_instance": cnt.value / args.count}), flush=True)


if __name__ == "__main__":
    main()
