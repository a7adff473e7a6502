"""Spectrum text files (reference
``pkg/src/fps_sft/core.py:280-333``, ``save_spectrum`` / ``load_spectrum``):
a ``# shape N_0 ... N_{D-1}`` header, then one ``m_0 ... m_{D-1} re im`` line
per entry, amplitudes with 17 significant digits (doubles round-trip
exactly).  Other ``#`` lines and blank lines are ignored.  Parse errors are
``ValueError("<path>:<line>: ...")`` with the reference's wording.

``save_batch`` writes one file per instance of a ``BatchResult`` (the
device output of ``fps_sft_batch``), ``load_batch`` reads files back into
the padded device layout that ``ops.synthesize`` / ``fpssft_synthesize``
consume."""

from __future__ import annotations

import os

import numpy as np

from .core import CubeShape, SparseSpectrum


def _format(spectrum: SparseSpectrum) -> str:
    lines = ["# shape " + " ".join(map(str, spectrum.shape.dims))]
    for freq, amp in spectrum.entries.items():
        lines.append(" ".join(map(str, freq)) + f" {amp.real:.17g} {amp.imag:.17g}")
    return "\n".join(lines) + "\n"


def save_spectrum(spectrum: SparseSpectrum, path) -> None:
    with open(path, "w", encoding="ascii") as fh:
        fh.write(_format(spectrum))


def _parse_entry(fields, shape: CubeShape, where: str):
    if len(fields) != shape.ndim + 2:
        raise ValueError(f"{where}: expected {shape.ndim + 2} fields, got {len(fields)}")
    try:
        freq = tuple(int(v) for v in fields[:-2])
        amp = complex(float(fields[-2]), float(fields[-1]))
    except ValueError as exc:
        raise ValueError(f"{where}: {exc}") from None
    if not shape.contains(freq):
        raise ValueError(f"{where}: index {freq} out of range {shape.dims}")
    if amp == 0:
        raise ValueError(f"{where}: zero amplitude")
    return freq, amp


def load_spectrum(path) -> SparseSpectrum:
    shape = None
    entries: dict = {}
    with open(path, "r", encoding="ascii") as fh:
        for no, raw in enumerate(fh, start=1):
            text = raw.strip()
            where = f"{path}:{no}"
            if not text:
                continue
            if text[0] == "#":
                words = text[1:].split()
                if words and words[0] == "shape":
                    if shape is not None:
                        raise ValueError(f"{where}: duplicate shape header")
                    try:
                        shape = CubeShape(tuple(int(v) for v in words[1:]))
                    except ValueError as exc:
                        raise ValueError(f"{where}: bad shape header: {exc}") from None
                continue
            if shape is None:
                raise ValueError(f"{where}: entry before '# shape' header")
            freq, amp = _parse_entry(text.split(), shape, where)
            if freq in entries:
                raise ValueError(f"{where}: duplicate frequency {freq}")
            entries[freq] = amp
    if shape is None:
        raise ValueError(f"{path}: missing '# shape' header")
    return SparseSpectrum(shape, entries)


def save_batch(result, directory, stem: str = "spectrum") -> list:
    """One text file per instance of a ``BatchResult``; returns the paths."""
    os.makedirs(directory, exist_ok=True)
    paths = []
    for b in range(result.batch):
        p = os.path.join(directory, f"{stem}_{b:06d}.txt")
        save_spectrum(result.report(b).recovered, p)
        paths.append(p)
    return paths


def load_batch(paths, device=None, k_cap: int | None = None):
    """Spectrum files -> (freqs [B, k_cap, D] int32, amps [B, k_cap]
    complex128, counts [B] int32) CUDA tensors, the layout of
    ``BatchResult`` and of ``ops.synthesize``.  All files must share a shape."""
    import torch

    specs = [load_spectrum(p) for p in paths]
    if not specs:
        raise ValueError("no spectrum files")
    shape = specs[0].shape
    if any(s.shape != shape for s in specs):
        raise ValueError("spectrum files have different shapes")
    kmax = max(1, max(len(s) for s in specs))
    k_cap = k_cap or 1 << (kmax - 1).bit_length()
    if k_cap < kmax:
        raise ValueError(f"k_cap {k_cap} below the largest file ({kmax} entries)")
    f = np.zeros((len(specs), k_cap, shape.ndim), np.int32)
    a = np.zeros((len(specs), k_cap), np.complex128)
    c = np.zeros(len(specs), np.int32)
    for b, s in enumerate(specs):
        n = len(s)
        c[b] = n
        if n:
            f[b, :n] = s.freq_array
            a[b, :n] = s.amp_array
    dev = torch.device(device if device is not None else "cuda")
    return (torch.as_tensor(f, device=dev), torch.as_tensor(a, device=dev),
            torch.as_tensor(c, device=dev), shape)
