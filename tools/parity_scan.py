#!/usr/bin/env python
"""Parity of the device path on exactly the cubes bench.py generates (its
make_spectra + on-device synthesis), instance by instance against the CPU
oracle: prints one JSON line per (config, precision) and, for every
instance that differs, its per-iteration (candidates, accepted, rejected)
logs on both sides and the symmetric support difference.

usage: tools/parity_scan.py --config 4 --count 512 [--precisions fp32,fp32-guarded]"""
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
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--count", type=int, default=512)
    ap.add_argument("--precisions", default="fp32")
    ap.add_argument("--k-cap", type=int, default=0)
    args = ap.parse_args()
    import numpy as np
    import torch

    import bench
    import paper_1711_11407_b200 as P
    from paper_1711_11407_b200 import workloads as W

    global _JOB
    c = args.config
    w = W.CONFIGS[c]
    dev = torch.device("cuda:0")
    spectra = W.make_spectra(w, args.count, 0)
    cubes = W.synthesize_batch_torch(w.dims, spectra, dev, w.noise_var,
                                     noise_seed=w.seed * 1000003)
    host = cubes.cpu().numpy()
    _JOB = (host, w.dims, P.PROFILES[w.profile], c)
    with get_context("fork").Pool(os.cpu_count()) as pool:
        refs = pool.map(_oracle, range(len(host)))
    for prec in args.precisions.split(","):
        cfg = P.FpsSftConfig(seed=c, **P.PROFILES[w.profile])
        k_cap = args.k_cap or bench.K_CAP[c]
        res = P.fps_sft_batch(cubes, cfg, k_cap=k_cap, precision=prec, iter_stats=True)
        bad = []
        same = 0
        worst = 0.0
        for b, ref in enumerate(refs):
            rep = res.report(b)
            got = {tuple(f) for f in rep.recovered.freq_array.tolist()}
            want = {tuple(f) for f in ref.freqs.tolist()}
            glog = [(s.candidates, s.accepted, s.rejected) for s in rep.iteration_log]
            wlog = [tuple(int(v) for v in x[2:]) for x in ref.log]
            ok = (got == want and glog == wlog and rep.iterations_run == ref.iterations_run
                  and rep.terminated_by == ref.terminated_by)
            if got == want and len(ref.amps):
                worst = max(worst, float(np.max(np.abs(rep.recovered.amp_array - ref.amps)
                                                / np.abs(ref.amps))))
            if ok:
                same += 1
            else:
                bad.append({"instance": b, "sym_diff": sorted(got ^ want)[:6],
                            "gpu": [rep.iterations_run, rep.terminated_by, glog],
                            "oracle": [ref.iterations_run, ref.terminated_by, wlog]})
        print(json.dumps({"config": c, "precision": prec, "instances": len(refs),
                          "identical": same, "max_rel_amp_err_on_identical_support": worst,
                          "differing": bad[:10]}), flush=True)


if __name__ == "__main__":
    main()
