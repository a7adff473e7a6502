"""Host-side line schedule: the (alpha_t, tau_t) sequence of one recovery.

The reference draws one slope and one offset per iteration from
``np.random.default_rng(config.seed)`` (driver.py:131, 142-143): the slope by
rejection sampling over the grid until it passes the Lemma-2 coprimality
test (numtheory.py:54-81, 95-110), the offset with ``rng.integers(0, dims)``.
The draws never depend on the data, so the whole schedule is a pure function
of ``(seed, shape)``: ``schedule_from_seed`` replays it with numpy's own
generator (same calls, same order), and the device loop consumes it as an
explicit int32 tensor [S, T, 2, D].  Pinned against the reference's draws by
``tests/test_host.py`` (golden ``ops.npz`` ``sched*`` arrays).
"""

from __future__ import annotations

import itertools
import math
from functools import lru_cache

import numpy as np

from .core import CubeShape

_REJECTION_CAP_FACTOR = 10  # numtheory.py:32-34
_ENUM_MAX = 2**22


def is_valid_slope(alpha, shape: CubeShape) -> bool:
    """Lemma 2, generalised to D (numtheory.py:54-81): over the active
    dimensions (N_k > 1) the alpha_k are pairwise coprime, coprime to every
    other dimension's cofactor, and gcd(L, c_k alpha_k ...) = 1."""
    alpha = tuple(int(a) for a in alpha)
    if len(alpha) != shape.ndim:
        raise ValueError(f"slope {alpha} has wrong dimensionality for {shape.dims}")
    for a, n in zip(alpha, shape.dims):
        if not 0 <= a < n:
            raise ValueError(f"slope component {a} out of range [0, {n})")
    return _valid(alpha, shape.dims)


@lru_cache(maxsize=1 << 16)
def _valid(alpha: tuple, dims: tuple) -> bool:
    L = math.lcm(*dims)
    cof = [L // n for n in dims]
    act = [k for k, n in enumerate(dims) if n > 1]
    for x, i in enumerate(act):
        if any(math.gcd(alpha[i], alpha[j]) != 1 for j in act[x + 1:]):
            return False
        if any(math.gcd(alpha[i], cof[j]) != 1 for j in act if j != i):
            return False
    g = L
    for k in act:
        g = math.gcd(g, cof[k] * alpha[k])
    return g == 1


def valid_slopes(shape: CubeShape) -> list[tuple[int, ...]]:
    if shape.n_total > _ENUM_MAX:
        raise ValueError(f"refusing to enumerate slopes for {shape.n_total} grid points")
    return [a for a in itertools.product(*(range(n) for n in shape.dims))
            if _valid(a, shape.dims)]


def sample_slope(shape: CubeShape, rng: np.random.Generator) -> tuple[int, ...]:
    """Uniform draw over the valid slopes, consuming ``rng`` exactly like
    numtheory.py:95-110 (rejection with a 10 N cap, then enumeration)."""
    dims = shape.dims_array
    for _ in range(_REJECTION_CAP_FACTOR * shape.n_total):
        alpha = tuple(int(a) for a in rng.integers(0, dims))
        if _valid(alpha, shape.dims):
            return alpha
    pool = valid_slopes(shape)
    return pool[int(rng.integers(0, len(pool)))]


def schedule_from_seed(shape: CubeShape, seed: int, t_max: int) -> np.ndarray:
    """int32 (t_max, 2, D): row t = (alpha_t, tau_t) of iteration t+1."""
    rng = np.random.default_rng(seed)
    out = np.empty((t_max, 2, shape.ndim), dtype=np.int32)
    for t in range(t_max):
        out[t, 0] = sample_slope(shape, rng)
        out[t, 1] = rng.integers(0, shape.dims_array)
    return out


_POOL = None


def _schedule_job(args):
    dims, seed, t_max = args
    return schedule_from_seed(CubeShape(dims), seed, t_max)


def schedules_from_seeds(shape: CubeShape, seeds, t_max: int, workers: int | None = None):
    """int32 (S, t_max, 2, D): ``schedule_from_seed`` for every seed (Monte
    Carlo trials each draw their own lines).  The replay is numpy's own
    generator call by call (~50 us per iteration), so many trials are spread
    over a pool of host processes (spawned: the parent may hold a CUDA
    context); small requests run in place."""
    import os

    seeds = [int(s) for s in seeds]
    if workers is None:
        workers = os.cpu_count() or 1
    if workers <= 1 or len(seeds) * t_max < 4000:
        return np.stack([schedule_from_seed(shape, s, t_max) for s in seeds]) if seeds else \
            np.empty((0, t_max, 2, shape.ndim), np.int32)
    global _POOL
    if _POOL is None:
        import multiprocessing as mp
        from concurrent.futures import ProcessPoolExecutor

        _POOL = ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("spawn"))
    jobs = [(shape.dims, s, t_max) for s in seeds]
    return np.stack(list(_POOL.map(_schedule_job, jobs, chunksize=max(1, len(jobs) // (4 * workers)))))


def bins_of_frequencies(freqs, alpha, shape: CubeShape) -> np.ndarray:
    """sum_k c_k alpha_k m_k mod L over a (K, D) array (numtheory.py:139-153)."""
    w = np.asarray([c * int(a) for c, a in zip(shape.cofactors, alpha)], dtype=np.int64)
    return (np.asarray(freqs, dtype=np.int64).reshape(-1, shape.ndim) @ w) % shape.line_len
