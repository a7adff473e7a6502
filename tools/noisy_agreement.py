#!/usr/bin/env python
"""Agreement of the device path with the CPU oracle on the noisy configs
(3 and 5, profile PN): per precision, the fraction of instances whose
recovered support is identical to the oracle's, the worst symmetric support
difference, and the largest relative amplitude error on identical supports.
Prints one JSON line per (config, precision)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="3,5")
    ap.add_argument("--count", type=int, default=64)
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_1711_11407_b200 as P
    from oracle import fps_oracle as O
    from paper_1711_11407_b200 import workloads as W

    for c in [int(x) for x in args.configs.split(",")]:
        w = W.CONFIGS[c]
        inst = [W.make_instance(w, r) for r in W.instance_rngs(w.seed, args.count)]
        cubes = torch.as_tensor(np.stack([x for _, _, x in inst])).cuda()
        prof = O.Profile(**P.PROFILES[w.profile])
        refs = [O.recover(x, w.dims, prof, seed=c) for _, _, x in inst]
        for prec in ("fp32", "fp64"):
            cfg = P.FpsSftConfig(seed=c, **P.PROFILES[w.profile])
            k_cap = 1024 if prec == "fp32" else min(1024, P.max_k_cap(P.CubeShape(w.dims), "fp64"))
            res = P.fps_sft_batch(cubes, cfg, k_cap=k_cap, precision=prec)
            same, worst, amp_err, iters_same = 0, 0, 0.0, 0
            for b, ref in enumerate(refs):
                rep = res.report(b)
                got = {tuple(f) for f in rep.recovered.freq_array.tolist()}
                want = {tuple(f) for f in ref.freqs.tolist()}
                if got == want:
                    same += 1
                    a = rep.recovered.amp_array
                    amp_err = max(amp_err, float(np.max(np.abs(a - ref.amps) / np.abs(ref.amps)))
                                  if len(a) else 0.0)
                    iters_same += rep.iterations_run == ref.iterations_run
                else:
                    worst = max(worst, len(got ^ want))
            print(json.dumps({"config": c, "precision": prec, "instances": len(refs),
                              "identical_support": same, "identical_iterations": iters_same,
                              "worst_symmetric_difference": worst,
                              "max_rel_amp_err_on_identical": amp_err,
                              "mean_k_oracle": float(np.mean([len(r.amps) for r in refs]))}),
                  flush=True)


if __name__ == "__main__":
    main()
