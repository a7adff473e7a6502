#!/usr/bin/env python
"""Agreement of the device path with the CPU oracle on the noisy configs
(3 and 5, profile PN), per precision: instances whose recovered support,
iteration count / termination and per-iteration (candidates, accepted,
rejected) log are identical to the oracle's, the worst symmetric support
difference, and the largest relative amplitude error on identical supports.
Prints one JSON line per (config, precision)."""
import argparse
import json
import os
import sys
from multiprocessing import get_context

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

_JOB = None


def _oracle(i):
    from oracle import fps_oracle as O

    cubes, dims, prof, seed = _JOB
    return O.recover(cubes[i], dims, O.Profile(**prof), seed=seed)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="3,5")
    ap.add_argument("--count", type=int, default=64)
    ap.add_argument("--start", type=int, default=0)
    ap.add_argument("--precisions", default="fp32,fp32-guarded,fp64")
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_1711_11407_b200 as P
    from paper_1711_11407_b200 import workloads as W

    global _JOB
    for c in [int(x) for x in args.configs.split(",")]:
        w = W.CONFIGS[c]
        inst = [W.make_instance(w, r) for r in W.instance_rngs(w.seed, args.count, args.start)]
        host = np.stack([x for _, _, x in inst])
        cubes = torch.as_tensor(host).cuda()
        _JOB = (host, w.dims, P.PROFILES[w.profile], c)
        with get_context("fork").Pool(os.cpu_count()) as pool:
            refs = pool.map(_oracle, range(len(inst)))
        for prec in args.precisions.split(","):
            cfg = P.FpsSftConfig(seed=c, **P.PROFILES[w.profile])
            k_cap = 1024 if prec != "fp64" else min(1024, P.max_k_cap(P.CubeShape(w.dims), "fp64"))
            res = P.fps_sft_batch(cubes, cfg, k_cap=k_cap, precision=prec, iter_stats=True)
            same, worst, amp_err, iters_same, logs_same = 0, 0, 0.0, 0, 0
            first_div = []
            for b, ref in enumerate(refs):
                rep = res.report(b)
                got = {tuple(f) for f in rep.recovered.freq_array.tolist()}
                want = {tuple(f) for f in ref.freqs.tolist()}
                glog = [(s.candidates, s.accepted, s.rejected) for s in rep.iteration_log]
                wlog = [tuple(int(v) for v in x[2:]) for x in ref.log]
                logs_same += glog == wlog
                if glog != wlog:
                    d = next((t for t, (x, y) in enumerate(zip(glog, wlog)) if x != y),
                             min(len(glog), len(wlog)))
                    first_div.append((b, d + 1))
                if got == want:
                    same += 1
                    a = rep.recovered.amp_array
                    amp_err = max(amp_err, float(np.max(np.abs(a - ref.amps) / np.abs(ref.amps)))
                                  if len(a) else 0.0)
                    iters_same += (rep.iterations_run == ref.iterations_run
                                   and rep.terminated_by == ref.terminated_by)
                else:
                    worst = max(worst, len(got ^ want))
            print(json.dumps({"config": c, "precision": prec, "instances": len(refs),
                              "first_instance": args.start,
                              "identical_support": same, "identical_iterations": iters_same,
                              "identical_logs": logs_same,
                              "worst_symmetric_difference": worst,
                              "max_rel_amp_err_on_identical": amp_err,
                              "first_log_divergence": first_div[:8],
                              "mean_k_oracle": float(np.mean([len(r.amps) for r in refs]))}),
                  flush=True)


if __name__ == "__main__":
    main()
