"""Golden fixtures for the imaging duality path, from the UNMODIFIED reference.

Run in the build container (the reference exists only there):

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src:. \
        python tests/golden/make_imaging_golden.py

Records what ``fps_sft.imaging`` returns (``reconstruct_sparse_image``,
imaging.py:104-143; ``synthetic_phantom`` / ``sparsify`` /
``threshold_for_fraction``, imaging.py:56-101):

* small pixel-sparse images (seeded here), stored verbatim with the
  reference's recovered entries, iterations, samples and reconstruction;
* phantom pins: SHA-256 of ``synthetic_phantom`` at small and full size and
  of the sparsified 512x576 images at the paper's three sparsity levels;
* the 512x576 duality runs (``FpsSftConfig(stall_limit=10, seed=800+level)``,
  the paper's Fig. 3 setting): K, iterations, samples, percent of frequency
  samples, termination, max pixel error, and the reference's wall time.

Output: ``tests/golden/imaging.npz`` + ``tests/golden/imaging.json``.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from fps_sft.driver import FpsSftConfig  # noqa: E402
from fps_sft.imaging import (GrayImage, nonzero_fraction, reconstruct_sparse_image,  # noqa: E402
                             sparsify, synthetic_phantom, threshold_for_fraction)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def small_cases():
    rng = np.random.default_rng(4242)
    out = []
    for dims in ((4, 4), (8, 8), (8, 12), (16, 16), (12, 18)):
        for t in range(4):
            k = int(rng.integers(1, 7))
            flat = rng.choice(dims[0] * dims[1], size=k, replace=False)
            px = np.zeros(dims)
            for f in flat:
                px[np.unravel_index(int(f), dims)] = rng.uniform(0.05, 1.0)
            seed = int(rng.integers(0, 2**31))
            out.append((f"img_{dims[0]}x{dims[1]}_{t}", px,
                        dict(max_iterations=40, stall_limit=10, seed=seed)))
    # the reference's own single-pixel cases (test_imaging.py:140-155)
    for name, dims, pix, seed in (("one_4x4", (4, 4), {(1, 3): 0.8}, 0),
                                  ("origin_8x8", (8, 8), {(0, 0): 1.0}, 1),
                                  ("offset_8x8", (8, 8), {(2, 3): 0.6}, 2)):
        px = np.zeros(dims)
        for p, v in pix.items():
            px[p] = v
        out.append((name, px, dict(max_iterations=8, seed=seed)))
    return out


def main():
    arrays, meta = {}, {"small": [], "phantom": {}, "duality_512x576": []}
    for name, px, cfg in small_cases():
        recon, rep = reconstruct_sparse_image(GrayImage(px), FpsSftConfig(**cfg))
        keys = list(rep.recovered.entries)
        arrays[f"{name}/pixels"] = px
        arrays[f"{name}/recon"] = recon.pixels
        arrays[f"{name}/freqs"] = np.asarray(keys, np.int64).reshape(-1, 2)
        arrays[f"{name}/amps"] = np.asarray([rep.recovered.entries[k] for k in keys], np.complex128)
        meta["small"].append(dict(name=name, cfg=cfg, iterations_run=rep.iterations_run,
                                  samples_used=rep.samples_used,
                                  terminated_by=rep.terminated_by))
        print(name, rep.iterations_run, rep.terminated_by, len(keys), flush=True)
    for dims, seed in (((32, 48), 2), ((64, 72), 5)):
        meta["phantom"][f"{dims[0]}x{dims[1]}_s{seed}"] = sha(synthetic_phantom(dims, seed).pixels)
    phantom = synthetic_phantom((512, 576), seed=1)
    meta["phantom"]["512x576_s1"] = sha(phantom.pixels)
    for level, target in enumerate((0.0285, 0.0448, 0.0661)):
        thr = threshold_for_fraction(phantom, target)
        sparse = sparsify(phantom, thr)
        cfg = dict(stall_limit=10, seed=800 + level)
        t0 = time.perf_counter()
        recon, rep = reconstruct_sparse_image(sparse, FpsSftConfig(**cfg))
        wall = time.perf_counter() - t0
        err = float(np.abs(recon.pixels - sparse.pixels).max())
        row = dict(level=level, target=target, threshold=thr, sparse_sha=sha(sparse.pixels),
                   k=int(np.count_nonzero(sparse.pixels)), fraction=nonzero_fraction(sparse),
                   cfg=cfg, iterations_run=rep.iterations_run, samples_used=rep.samples_used,
                   percent_samples=rep.percent_samples(), terminated_by=rep.terminated_by,
                   recovered=len(rep.recovered.entries), max_pixel_error=err,
                   reference_wall_s=wall)
        meta["duality_512x576"].append(row)
        print(row, flush=True)
        np.savez_compressed(os.path.join(HERE, "imaging.npz"), **arrays)
        with open(os.path.join(HERE, "imaging.json"), "w") as fh:
            json.dump(meta, fh, indent=1)
    np.savez_compressed(os.path.join(HERE, "imaging.npz"), **arrays)
    with open(os.path.join(HERE, "imaging.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


if __name__ == "__main__":
    main()
