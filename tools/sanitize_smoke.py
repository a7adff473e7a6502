#!/usr/bin/env python
"""Small runs of every kernel family, for compute-sanitizer --tool memcheck
(warp static / warp runtime-shape / team / generic CTA kernels, per-step
kernels, synthesis)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1711_11407_b200 as P  # noqa: E402
from paper_1711_11407_b200 import ops  # noqa: E402
from paper_1711_11407_b200 import workloads as W  # noqa: E402

PROF = P.PROFILES["P32"]


def run(dims, k, B=3, k_cap=None, modes=("auto", "cta"), prec=("fp32", "fp64")):
    cubes = []
    for b in range(B):
        f, a = W.reference_generate(dims, k, 40 + b)
        cubes.append(W.synthesize_np(dims, f, a).astype(np.complex64))
    t = torch.as_tensor(np.stack(cubes)).cuda()
    cfg = P.FpsSftConfig(max_iterations=8, seed=3, **PROF)
    for mode in modes:
        for p in prec:
            kc = k_cap or (1 << max(4, (2 * k - 1).bit_length()))
            kc = min(kc, P.max_k_cap(P.CubeShape(dims), p, mode))
            try:
                res = P.fps_sft_batch(t, cfg, k_cap=kc, precision=p, mode=mode, iter_stats=True)
            except ValueError as e:
                print("skip", dims, mode, p, e)
                continue
            img = ops.synthesize(res)
            torch.cuda.synchronize()
            print(dims, mode, p, res.count.tolist(), res.terminated_by.tolist(), img.shape)


def run_group_and_guarded():
    """The group-gather kernel (interleaved batch, shared schedule) and the
    guarded float32 kernels (noisy profile: warp 64^3, team 512^2)."""
    w = W.CONFIGS[2]
    inst = [W.make_instance(w, r) for r in W.instance_rngs(w.seed, 8)]
    cubes = torch.as_tensor(np.stack([c for _, _, c in inst])).cuda()
    cfg = P.FpsSftConfig(seed=2, **PROF)
    r = P.BatchRunner(P.CubeShape(w.dims), cfg, 8, k_cap=128, device="cuda", group=8)
    res = r.run(P.interleave(cubes, 8))
    torch.cuda.synchronize()
    print("group kernel", r.plan, res.count.tolist())
    pn = P.PROFILES["PN"]
    for dims, k in (((64, 64, 64), 40), ((512, 512), 60)):
        cubes = []
        for b in range(2):
            f, a = W.reference_generate(dims, k, 70 + b)
            x = W.synthesize_np(dims, f, a)
            x = x + 0.05 * (np.random.default_rng(b).standard_normal(x.shape)
                            + 1j * np.random.default_rng(b + 9).standard_normal(x.shape))
            cubes.append(x.astype(np.complex64))
        t = torch.as_tensor(np.stack(cubes)).cuda()
        cfg = P.FpsSftConfig(max_iterations=6, seed=5, **pn)
        for mode in ("auto", "cta"):
            res = P.fps_sft_batch(t, cfg, k_cap=256, precision="fp32-guarded", mode=mode,
                                  iter_stats=True)
            torch.cuda.synchronize()
            print("guarded", dims, mode, res.count.tolist(), res.terminated_by.tolist())


if __name__ == "__main__":
    run_group_and_guarded()
    run((256, 256), 40)
    run((512, 512), 60, k_cap=128)
    run((1024, 2048), 50, B=2, k_cap=256)
    run((64, 64, 64), 30)
    run((12, 18), 9)
    run((16, 16), 12, k_cap=8)
    x = torch.randn(2, 60, dtype=torch.complex64).cuda()
    ops.dft_forward(x)
    ops.line_spectra(torch.zeros((1, 12, 18), dtype=torch.complex64).cuda(), (1, 1), (0, 0))
    ops.project_onto_bins(np.array([[1, 2]]), np.array([1 + 1j]), (1, 1), (0, 0), P.CubeShape((12, 18)))
    torch.cuda.synchronize()
    print("sanitize smoke done")
