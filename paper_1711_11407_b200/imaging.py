"""Sparse-image reconstruction through time/frequency duality on the GPU
(reference ``pkg/src/fps_sft/imaging.py:104-143``).

A pixel-sparse image is transformed once (dense 1/N D-D DFT, the reference's
``oracle.dense_dft``, ``oracle.py:36-43``; here cuFFT through torch, a
one-time input transform); the frequency cube is handed to the recovery
loop, and each recovered sinusoid (m, a) is the pixel at (-m mod N) with
value Re(a N).  The 512 x 576 images of the paper's Fig. 3 have
L = lcm(512, 576) = 4608 and up to ~20k pixels, so the loop is
``large.fps_sft_large`` (float64, global-memory lines and recovered set).

The image helpers mirror the reference's names and semantics
(``imaging.py:35-101``): ``GrayImage``, ``nonzero_fraction``, ``sparsify``,
``threshold_for_fraction`` and the deterministic ``synthetic_phantom``
(a sum of 40 random anisotropic Gaussian blobs under a super-Gaussian
elliptical window, normalised to [0, 1]; same draw order, so the same
pixels -- pinned by SHA-256 in tests/golden/imaging.json).  PGM I/O is not
part of this path.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np

from .core import CubeShape
from .driver import FpsSftConfig, RecoveryReport, default_max_iterations
from .large import fps_sft_large

IMAG_RESIDUE_TOL = 1e-8  # imaging.py:21


@dataclass(frozen=True)
class GrayImage:
    """Row-major (H, W) float image with values in [0, 1]."""

    pixels: np.ndarray

    def __post_init__(self):
        p = np.asarray(self.pixels, dtype=np.float64)
        if p.ndim != 2 or p.size == 0:
            raise ValueError("pixels must be a nonempty 2-D array")
        if p.min() < 0.0 or p.max() > 1.0:
            raise ValueError("pixel values must lie in [0, 1]")
        object.__setattr__(self, "pixels", p)

    @property
    def height(self) -> int:
        return self.pixels.shape[0]

    @property
    def width(self) -> int:
        return self.pixels.shape[1]


def nonzero_fraction(img: GrayImage) -> float:
    return np.count_nonzero(img.pixels) / img.pixels.size


def sparsify(img: GrayImage, threshold: float) -> GrayImage:
    """Pixels below ``threshold`` set to zero (``>=`` keeps)."""
    if not 0.0 <= threshold <= 1.0:
        raise ValueError("threshold must lie in [0, 1]")
    return GrayImage(np.where(img.pixels < threshold, 0.0, img.pixels))


def threshold_for_fraction(img: GrayImage, fraction: float) -> float:
    """The ``>=`` cut that keeps about ``fraction`` of the pixels."""
    if not 0.0 < fraction <= 1.0:
        raise ValueError("fraction must lie in (0, 1]")
    return float(np.quantile(img.pixels, 1.0 - fraction))


def synthetic_phantom(dims: tuple[int, int] = (512, 576), seed: int = 0) -> GrayImage:
    """Deterministic smooth test image (the reference's stand-in for the
    paper's MRI slice): 40 blobs with centre in [-0.75, 0.75]^2, widths in
    [0.03, 0.25], correlation in [-0.5, 0.5] and weight in [0.2, 1] drawn in
    that order per blob from default_rng(seed), on coordinates normalised to
    [-1, 1); times exp(-((y/0.9)^2 + (x/0.9)^2)^4 / 2); min-max normalised."""
    h, w = dims
    rng = np.random.default_rng(seed)
    rows, cols = np.mgrid[0:h, 0:w]
    y = (rows - h / 2) / (h / 2)
    x = (cols - w / 2) / (w / 2)
    acc = np.zeros((h, w))
    for _ in range(40):
        cy, cx = rng.uniform(-0.75, 0.75, size=2)
        sy, sx = rng.uniform(0.03, 0.25, size=2)
        rho = rng.uniform(-0.5, 0.5)
        weight = rng.uniform(0.2, 1.0)
        u = (y - cy) / sy
        v = (x - cx) / sx
        acc += weight * np.exp(-0.5 * (u**2 + v**2 - 2 * rho * u * v) / (1 - rho**2))
    acc *= np.exp(-0.5 * ((y / 0.9) ** 2 + (x / 0.9) ** 2) ** 4)
    acc -= acc.min()
    acc /= acc.max()
    return GrayImage(acc)


def dense_dft(pixels: np.ndarray, device=None):
    """Full D-D DFT with 1/N normalisation (oracle.py:36-43) on the device,
    complex128."""
    import torch

    dev = torch.device(device if device is not None else "cuda")
    x = torch.as_tensor(np.asarray(pixels, np.complex128), device=dev)
    if x.numel() == 0:
        raise ValueError("empty cube")
    return torch.fft.fftn(x) / x.numel()


def reconstruct_sparse_image(img_sparse: GrayImage, config: FpsSftConfig = FpsSftConfig(), *,
                             device=None, loop: str = "device") -> tuple[GrayImage, RecoveryReport]:
    """Recover a pixel-sparse image from samples of its frequency cube
    (imaging.py:104-143): absolute tolerances rescaled by 1/N, the iteration
    cap opened up from the pixel count when ``max_iterations`` is None, and
    each recovered (m, a) written to pixel (-m mod N) = Re(a N)."""
    shape = CubeShape(img_sparse.pixels.shape)
    n = shape.n_total
    k = int(np.count_nonzero(img_sparse.pixels))
    cfg = replace(config, amp_prune_tol=config.amp_prune_tol / n,
                  energy_floor_abs=config.energy_floor_abs / n)
    if cfg.max_iterations is None:
        cfg = replace(cfg, max_iterations=max(default_max_iterations(shape),
                                              math.ceil(4 * k / shape.line_len) + 20))
    xhat = dense_dft(img_sparse.pixels, device)
    report = fps_sft_large(xhat, shape, cfg, precision="fp64", loop=loop)
    out = np.zeros(shape.dims)
    freqs, values = report.recovered.freq_array, report.recovered.amp_array * n
    bad = np.flatnonzero(np.abs(values.imag) > IMAG_RESIDUE_TOL)
    if bad.size:
        i = int(bad[0])
        raise ValueError(f"non-real reconstructed pixel value {complex(values[i])!r} at dual "
                         f"index {tuple(int(v) for v in freqs[i])}")
    if len(freqs):
        out[tuple(((-freqs) % np.asarray(shape.dims)).T)] = values.real
    return GrayImage(np.clip(out, 0.0, 1.0)), report
