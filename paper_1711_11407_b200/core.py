"""Domain types of the FPS-SFT path, mirroring the reference's public ones.

Same names, argument meaning and error behaviour as ``fps_sft.core``
(``/root/reference/pkg/src/fps_sft/core.py``) for the subset the recovery
loop needs: ``CubeShape`` (:26-73), ``Sinusoid`` (:76-81), ``SparseSpectrum``
(:84-143), ``spectra_match`` (:146-157), ``SignalSource`` (:160-173),
``DenseSource``/``make_dense_source`` (:220-238, :276-278).

Difference by design: ``DenseSource`` keeps the cube as complex64 (the dtype
the device path reads from HBM) instead of upcasting to complex128
(core.py:224); a complex128 cube is rounded once on entry.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from functools import cached_property
from typing import Iterable, Mapping, Sequence

import numpy as np

INT64_SAFE = 2**62
FreqIndex = tuple[int, ...]


@dataclass(frozen=True)
class CubeShape:
    """Extents [N_0, ..., N_{D-1}]; derived N, L = lcm and c_k = L / N_k."""

    dims: tuple[int, ...]

    def __init__(self, dims: Iterable[int]):
        dims = tuple(int(n) for n in dims)
        if not dims:
            raise ValueError("shape needs at least one dimension")
        if min(dims) < 1:
            raise ValueError(f"dimension lengths must be >= 1, got {dims}")
        object.__setattr__(self, "dims", dims)

    @property
    def ndim(self) -> int:
        return len(self.dims)

    @cached_property
    def n_total(self) -> int:
        return math.prod(self.dims)

    @cached_property
    def line_len(self) -> int:
        L = math.lcm(*self.dims)
        if L >= INT64_SAFE:
            raise OverflowError(f"line length lcm{self.dims} exceeds the machine integer range")
        return L

    @cached_property
    def cofactors(self) -> tuple[int, ...]:
        return tuple(self.line_len // n for n in self.dims)

    @cached_property
    def dims_array(self) -> np.ndarray:
        return np.asarray(self.dims, dtype=np.int64)

    def contains(self, m: Sequence[int]) -> bool:
        return len(m) == self.ndim and all(0 <= int(v) < n for v, n in zip(m, self.dims))

    def validate_index(self, m: Sequence[int]) -> FreqIndex:
        m = tuple(int(v) for v in m)
        if not self.contains(m):
            raise ValueError(f"index {m} out of range for shape {self.dims}")
        return m


@dataclass(frozen=True)
class Sinusoid:
    amp: complex
    freq: FreqIndex


class SparseSpectrum:
    """Frequency tuple -> nonzero complex amplitude, kept in lexicographic order."""

    def __init__(self, shape: CubeShape, entries: Mapping[FreqIndex, complex]):
        self.shape = shape
        items = []
        for freq, amp in entries.items():
            freq = shape.validate_index(freq)
            amp = complex(amp)
            if amp == 0:
                raise ValueError(f"zero amplitude at frequency {freq}")
            if not (math.isfinite(amp.real) and math.isfinite(amp.imag)):
                raise ValueError(f"non-finite amplitude at frequency {freq}")
            items.append((freq, amp))
        items.sort(key=lambda kv: kv[0])
        if len({f for f, _ in items}) != len(items):
            raise ValueError("duplicate frequency entries")
        self.entries: dict[FreqIndex, complex] = dict(items)

    @classmethod
    def _trusted(cls, shape: CubeShape, freqs: np.ndarray, amps: np.ndarray) -> "SparseSpectrum":
        """Build from device output already validated, sorted and unique."""
        self = cls.__new__(cls)
        self.shape = shape
        freqs = np.asarray(freqs, np.int64).reshape(-1, shape.ndim)
        amps = np.asarray(amps, np.complex128).reshape(-1)
        self.__dict__["_entries"] = None  # the dict is built on first use (large sets)
        self.__dict__["freq_array"] = freqs  # cached_property values, already at hand
        self.__dict__["amp_array"] = amps
        return self

    @property
    def entries(self) -> dict:
        e = self.__dict__.get("_entries")
        if e is None:
            e = dict(zip(map(tuple, self.freq_array.tolist()), self.amp_array.tolist()))
            self.__dict__["_entries"] = e
        return e

    @entries.setter
    def entries(self, value) -> None:
        self.__dict__["_entries"] = value

    @classmethod
    def from_sinusoids(cls, shape: CubeShape, sinusoids: Iterable[Sinusoid]) -> "SparseSpectrum":
        return cls(shape, {s.freq: s.amp for s in sinusoids})

    @property
    def k(self) -> int:
        return len(self.entries)

    def __len__(self) -> int:
        return len(self.entries)

    def __eq__(self, other) -> bool:
        return (isinstance(other, SparseSpectrum) and self.shape == other.shape
                and self.entries == other.entries)

    def __repr__(self) -> str:
        return f"SparseSpectrum(shape={self.shape.dims}, k={self.k})"

    @cached_property
    def freq_array(self) -> np.ndarray:
        if not self.entries:
            return np.zeros((0, self.shape.ndim), dtype=np.int64)
        return np.asarray(list(self.entries.keys()), dtype=np.int64)

    @cached_property
    def amp_array(self) -> np.ndarray:
        return np.asarray(list(self.entries.values()), dtype=np.complex128)

    def scaled(self, factor: complex) -> "SparseSpectrum":
        if factor == 0:
            raise ValueError("scale factor must be nonzero")
        return SparseSpectrum(self.shape, {f: a * factor for f, a in self.entries.items()})


def spectra_match(estimate: SparseSpectrum, truth: SparseSpectrum, rtol: float = 1e-8) -> bool:
    """Same key set and |est - true| <= rtol |true| for every entry."""
    if estimate.shape.dims != truth.shape.dims:
        return False
    if estimate.entries.keys() != truth.entries.keys():
        return False
    return all(abs(estimate.entries[f] - a) <= rtol * abs(a) for f, a in truth.entries.items())


class SignalSource:
    """Sample oracle n -> x(n).  The device path needs the dense cube, so a
    source is usable by ``fps_sft`` if it is a ``DenseSource`` or can evaluate
    ``sample_many`` on the whole grid (see ``driver.materialize``)."""

    def shape(self) -> CubeShape:  # pragma: no cover - interface
        raise NotImplementedError

    def sample(self, n: Sequence[int]) -> complex:  # pragma: no cover - interface
        raise NotImplementedError

    def sample_many(self, indices: np.ndarray) -> np.ndarray:
        return np.asarray([self.sample(row) for row in indices], dtype=np.complex128)


class DenseSource(SignalSource):
    """A materialised complex64 cube (numpy array or CUDA tensor)."""

    def __init__(self, cube, shape: CubeShape):
        dims = tuple(int(d) for d in getattr(cube, "shape", ()))
        if dims != shape.dims:
            raise ValueError(f"cube extents {dims} do not match shape {shape.dims}")
        if isinstance(cube, np.ndarray):
            cube = np.ascontiguousarray(cube, dtype=np.complex64)
        self._data = cube
        self._cube = shape

    @property
    def data(self):
        return self._data

    def shape(self) -> CubeShape:
        return self._cube

    def sample(self, n: Sequence[int]) -> complex:
        return complex(self._data[self._cube.validate_index(n)])

    def sample_many(self, indices: np.ndarray) -> np.ndarray:
        indices = np.asarray(indices, dtype=np.int64)
        data = self._data
        if not isinstance(data, np.ndarray):
            data = data.cpu().numpy()
        return data[tuple(indices.T)].astype(np.complex128)


def make_dense_source(cube, shape: CubeShape) -> DenseSource:
    """Sample oracle backed by a stored cube (core.py:276-278)."""
    return DenseSource(cube, shape)


class SyntheticSource(SignalSource):
    """Lazy sinusoid mixture x(n) = sum_i a_i exp(2j pi sum_k n_k m_ik / N_k)
    (reference ``SyntheticSource``, core.py:176-217): samples on the host
    with the same exact integer phases (multiples of 1/L of a turn); the
    device path materialises the whole grid with ``fpssft_synthesize``
    through ``spectrum`` (``driver.materialize``)."""

    def __init__(self, spectrum: SparseSpectrum):
        self.spectrum = spectrum
        self._cube = spectrum.shape

    def shape(self) -> CubeShape:
        return self._cube

    def sample(self, n: Sequence[int]) -> complex:
        return complex(self.sample_many(np.asarray([self._cube.validate_index(n)]))[0])

    def sample_many(self, indices: np.ndarray) -> np.ndarray:
        sh = self._cube
        idx = np.asarray(indices, dtype=np.int64).reshape(-1, sh.ndim)
        f = self.spectrum.freq_array
        a = self.spectrum.amp_array
        L = sh.line_len
        cof = np.asarray([L // d for d in sh.dims], np.int64)
        u = ((idx * cof) @ f.T) % L  # [n, K] exact phase numerators
        roots = np.exp(2j * np.pi * np.arange(L) / L)
        return (roots[u] * a[None, :]).sum(axis=1)


def make_synthetic_source(spec: SparseSpectrum) -> SyntheticSource:
    """Sample oracle evaluating the mixture lazily (core.py:270-273)."""
    return SyntheticSource(spec)
