"""Seeded synthetic workloads for the five BASELINE.json configs.

BASELINE.json names no dataset, so every input is synthetic (SURVEY.md
section 8(d)).  A workload is a batch of sparse spectra (integer frequency
tuples + complex amplitudes) and the complex64 cubes they synthesise to:

    x(n) = sum_i a_i exp(+2 pi j sum_k n_k m_ik / N_k)

built as an N-scaled inverse FFT in float64 and rounded once to complex64,
plus optional complex white Gaussian noise.  Instance ``b`` of a config draws
from ``np.random.default_rng(SeedSequence(seed).spawn(B)[b])`` the way the
reference derives per-trial seeds (``pkg/src/fps_sft/oracle.py:215-227``).

Uniform unit-magnitude draws follow the reference generator's draw order
(``oracle.py:88-99,129-139``: ``rng.choice(N, K, replace=False)`` then
``rng.uniform(0, 2 pi, K)``), so ``draw_spectrum`` on ``default_rng(s)``
returns the spectrum of ``generate(GeneratorSpec(shape, k, seed=s))``
(``reference_generate`` below; pinned by tests/test_oracle_golden.py).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    dims: tuple[int, ...]
    batch: int
    k: int
    placement: str  # "uniform" | "blobs"
    magnitude: str  # "unit" | "uniform_0.5_1.5" | "rayleigh"
    noise_var: float  # complex noise variance per sample (0 = noiseless)
    profile: str  # "P32" | "PN"
    seed: int


CONFIGS = {
    1: Workload("cfg1_256x256_k20", (256, 256), 1, 20, "uniform", "unit", 0.0, "P32", 101),
    2: Workload("cfg2_256x256_k100_b4096", (256, 256), 4096, 100, "uniform",
                "uniform_0.5_1.5", 0.0, "P32", 202),
    3: Workload("cfg3_64x64x64_k200_b1024_10dB", (64, 64, 64), 1024, 200, "uniform", "unit",
                0.1, "PN", 303),
    4: Workload("cfg4_1024x2048_k1000_b512_blobs", (1024, 2048), 512, 1000, "blobs",
                "rayleigh", 0.0, "P32", 404),
    5: Workload("cfg5_512x512_k500_b16384_20dB", (512, 512), 16384, 500, "uniform",
                "rayleigh", 0.02, "PN", 505),
}


def instance_rngs(seed: int, count: int, start: int = 0) -> list[np.random.Generator]:
    kids = np.random.SeedSequence(seed).spawn(start + count)[start:]
    return [np.random.default_rng(k) for k in kids]


def _uniform_support(rng, dims, k):
    flat = rng.choice(math.prod(dims), size=k, replace=False)
    return np.stack(np.unravel_index(flat, dims), axis=-1).astype(np.int64)


def _blob_support(rng, dims, k, n_blobs=10, std=8.0):
    """k distinct frequencies in ``n_blobs`` Gaussian blobs on the torus
    (config 4): centre uniform, offset rint(N(0, std^2)) per dim, duplicates
    redrawn."""
    dims_a = np.asarray(dims, np.int64)
    centres = rng.integers(0, dims_a, size=(n_blobs, len(dims)))
    seen: set[tuple[int, ...]] = set()
    out = []
    while len(out) < k:
        c = centres[int(rng.integers(0, n_blobs))]
        f = tuple(int(v) for v in (np.rint(c + rng.normal(0.0, std, len(dims))).astype(np.int64)
                                   % dims_a))
        if f not in seen:
            seen.add(f)
            out.append(f)
    return np.asarray(out, np.int64)


def draw_spectrum(w: Workload, rng: np.random.Generator):
    """(freqs (K, D) int64, amps (K,) complex128) for one instance."""
    if w.placement == "uniform":
        freqs = _uniform_support(rng, w.dims, w.k)
    else:
        freqs = _blob_support(rng, w.dims, w.k)
    if w.magnitude == "unit":
        mags = np.ones(w.k)
    elif w.magnitude == "uniform_0.5_1.5":
        mags = rng.uniform(0.5, 1.5, w.k)
    else:
        mags = rng.rayleigh(1.0, w.k)
    phases = rng.uniform(0.0, 2 * np.pi, size=w.k)
    amps = mags * (np.cos(phases) + 1j * np.sin(phases))
    return freqs, amps


def synthesize_np(dims, freqs, amps) -> np.ndarray:
    """complex128 cube of a sparse spectrum (inverse FFT scaled by N)."""
    grid = np.zeros(tuple(dims), np.complex128)
    np.add.at(grid, tuple(np.asarray(freqs, np.int64).T), np.asarray(amps, np.complex128))
    return np.fft.ifftn(grid) * math.prod(dims)


def reference_generate(dims, k: int, seed: int):
    """Spectrum of the reference's ``generate(GeneratorSpec(shape=dims, k=k,
    seed=seed))`` (uniform placement, unit magnitude)."""
    w = Workload("ref", tuple(dims), 1, k, "uniform", "unit", 0.0, "P64", seed)
    return draw_spectrum(w, np.random.default_rng(seed))


def make_instance(w: Workload, rng: np.random.Generator):
    """One instance on the host: (freqs, amps, complex64 cube)."""
    freqs, amps = draw_spectrum(w, rng)
    cube = synthesize_np(w.dims, freqs, amps)
    if w.noise_var > 0:
        s = math.sqrt(w.noise_var / 2)
        cube = cube + s * (rng.standard_normal(cube.shape) + 1j * rng.standard_normal(cube.shape))
    return freqs, amps, cube.astype(np.complex64)


def make_spectra(w: Workload, count: int | None = None, start: int = 0):
    """Spectra only (cheap) for instances [start, start+count)."""
    count = w.batch if count is None else count
    return [draw_spectrum(w, r) for r in instance_rngs(w.seed, count, start)]


def synthesize_batch_torch(dims, spectra, device, noise_var=0.0, noise_seed=0, out=None):
    """Device-side batch synthesis for the big configs (untimed data
    generation; cuFFT is used here only to build inputs).  Returns a
    complex64 tensor [B, *dims] on ``device``.  Noise comes from a torch
    generator seeded with ``noise_seed`` (deterministic for a given device
    type and chunking)."""
    import torch

    dims = tuple(int(d) for d in dims)
    B = len(spectra)
    if out is None:
        out = torch.empty((B, *dims), dtype=torch.complex64, device=device)
    N = math.prod(dims)
    chunk = max(1, min(B, (1 << 28) // (N * 16)))
    gen = torch.Generator(device=device)
    gen.manual_seed(int(noise_seed))
    for s in range(0, B, chunk):
        e = min(B, s + chunk)
        lin = np.concatenate([np.ravel_multi_index(tuple(np.asarray(f).T), dims) + j * N
                              for j, (f, _) in enumerate(spectra[s:e])])
        amp = np.concatenate([np.asarray(a, np.complex128) for _, a in spectra[s:e]])
        grid = torch.zeros((e - s) * N, dtype=torch.complex128, device=device)
        grid.index_put_((torch.as_tensor(lin, device=device),),
                        torch.as_tensor(amp, device=device), accumulate=True)
        grid = grid.view(e - s, *dims)
        cube = torch.fft.ifftn(grid, dim=tuple(range(1, len(dims) + 1))) * N
        del grid
        if noise_var > 0:
            sd = math.sqrt(noise_var / 2)
            nz = torch.randn((2, *cube.shape), dtype=torch.float64, device=device, generator=gen)
            cube += torch.complex(nz[0], nz[1]) * sd
            del nz
        out[s:e].copy_(cube)
        del cube
    return out
