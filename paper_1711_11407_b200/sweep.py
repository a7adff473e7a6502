"""Monte Carlo recovery sweeps on the GPU.

The reference measures recovery probability and sample budgets with
``run_sweep`` (``pkg/src/fps_sft/oracle.py:235-303``): for every (shape, K,
placement) cell it draws ``trials`` sparse spectra (``generate``,
``oracle.py:88-139``), runs ``fps_sft`` on each with its own seed, and
counts exact recoveries (``spectra_match``).  Here every cell is one batched
launch: the spectra are drawn on the host with the reference's draw order,
synthesised on the device (``fpssft_synthesize``), recovered with one
schedule per trial (``sched_index``), and matched against the truth.

Differences: the cubes are complex64 and the loop runs in ``precision``
(float32 by default), so the default profile is P32 and the match tolerance
is 1e-4 relative (the reference uses exact complex128 sources, default
tolerances and rtol=1e-8).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np

from .core import CubeShape
from .driver import PROFILES, FpsSftConfig, default_max_iterations, fps_sft_batch
from .schedule import schedules_from_seeds

CLUSTER_SIZES = {9: 1, 25: 2}  # cluster size -> block radius (oracle.py:31)
PLACEMENTS = {"uniform": ("uniform", None), "clustered9": ("clustered", 9),
              "clustered25": ("clustered", 25)}
SWEEP_COLUMNS = ("algo", "N0", "N1", "K", "placement", "trials", "p_success",
                 "mean_percent_samples", "mean_iters", "mean_wall_ms")


def trial_seeds(seed: int, n: int) -> list[tuple[int, int]]:
    """(generator seed, algorithm seed) per trial, derived like the
    reference (``oracle.py:215-227``): SeedSequence(seed).spawn(n), each child
    spawning one sequence for the generator and one for the algorithm."""
    out = []
    for child in np.random.SeedSequence(seed).spawn(n):
        g, a = child.spawn(2)
        out.append((int(g.generate_state(1, dtype=np.uint64)[0]),
                    int(a.generate_state(1, dtype=np.uint64)[0])))
    return out


def draw_support(shape: CubeShape, k: int, placement: str, cluster_size, rng) -> np.ndarray:
    """Frequency support in the reference's draw order (``oracle.py:88-126``):
    uniform without replacement, or disjoint square blocks of 9 / 25 with
    toroidal wrap, centres drawn as flat grid indices."""
    if placement == "uniform":
        flat = rng.choice(shape.n_total, size=k, replace=False)
        return np.stack(np.unravel_index(flat, shape.dims), axis=-1).astype(np.int64)
    radius = CLUSTER_SIZES[cluster_size]
    deltas = [(d0, d1) for d0 in range(-radius, radius + 1) for d1 in range(-radius, radius + 1)]
    taken: set = set()
    out = []
    for _ in range(k // cluster_size):
        for _attempt in range(10_000):
            c0, c1 = (int(v) for v in np.unravel_index(int(rng.integers(0, shape.n_total)),
                                                       shape.dims))
            block = [((c0 + a) % shape.dims[0], (c1 + b) % shape.dims[1]) for a, b in deltas]
            if len(set(block)) == cluster_size and not taken.intersection(block):
                taken.update(block)
                out.extend(block)
                break
        else:
            raise ValueError(f"could not place {k // cluster_size} disjoint clusters")
    return np.asarray(out, np.int64)


def generate_spectrum(shape: CubeShape, k: int, seed: int, placement: str = "uniform",
                      cluster_size=None, amp_magnitude: float = 1.0):
    """(freqs [K, D], amps [K]) of ``generate(GeneratorSpec(...))``
    (``oracle.py:129-139``): support, then uniform phases, fixed magnitude."""
    rng = np.random.default_rng(seed)
    freqs = draw_support(shape, k, placement, cluster_size, rng)
    ph = rng.uniform(0.0, 2 * np.pi, size=len(freqs))
    return freqs, amp_magnitude * (np.cos(ph) + 1j * np.sin(ph))


@dataclass(frozen=True)
class SweepRow:
    algo: str
    n0: int
    n1: int
    k: int
    placement: str
    trials: int
    p_success: float
    mean_percent_samples: float
    mean_iters: float
    mean_wall_ms: float

    def as_dict(self) -> dict:
        return dict(zip(SWEEP_COLUMNS, (self.algo, self.n0, self.n1, self.k, self.placement,
                                        self.trials, self.p_success, self.mean_percent_samples,
                                        self.mean_iters, self.mean_wall_ms)))


def run_cell(shape: CubeShape, k: int, placement: str, trials: int, seed: int,
             config: FpsSftConfig, *, precision: str = "fp32", match_rtol: float = 1e-4,
             device=None) -> tuple[SweepRow, dict]:
    """One sweep cell as one batched launch; returns the row and per-trial data."""
    import time

    import torch

    from . import ops

    dev = torch.device(device if device is not None else "cuda")
    kind, csize = PLACEMENTS[placement]
    seeds = trial_seeds(seed, trials)
    t_max = config.max_iterations or default_max_iterations(shape)
    truths = [generate_spectrum(shape, k, g, kind, csize) for g, _ in seeds]
    sched = schedules_from_seeds(shape, [a for _, a in seeds], t_max)
    k_in = 1 << max(0, (k - 1).bit_length())
    fr = torch.zeros((trials, k_in, shape.ndim), dtype=torch.int32)
    am = torch.zeros((trials, k_in), dtype=torch.complex128)
    for b, (f, a) in enumerate(truths):
        fr[b, :len(f)] = torch.as_tensor(f, dtype=torch.int32)
        am[b, :len(a)] = torch.as_tensor(a)
    cnt = torch.full((trials,), k, dtype=torch.int32)
    cubes = ops.synthesize(fr.to(dev), am.to(dev), cnt.to(dev), shape=shape, precision="fp64")
    k_cap = 1 << max(6, (2 * k - 1).bit_length())
    cfg = replace(config, max_iterations=t_max)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    res = fps_sft_batch(cubes, cfg, schedule=sched, sched_index=np.arange(trials),
                        k_cap=k_cap, precision=precision)
    torch.cuda.synchronize(dev)
    wall_ms = (time.perf_counter() - t0) * 1e3 / trials
    count = res.count.cpu().numpy()
    freqs = res.freqs.cpu().numpy()
    amps = res.amps.cpu().numpy()
    samples = res.samples_used.cpu().numpy()
    iters = res.iterations.cpu().numpy()
    ok = np.zeros(trials, bool)
    for b, (f, a) in enumerate(truths):
        if count[b] != len(f):
            continue
        order = np.lexsort(f.T[::-1])
        ok[b] = bool(np.array_equal(freqs[b, :count[b]], f[order]) and
                     np.all(np.abs(amps[b, :count[b]] - a[order]) <= match_rtol * np.abs(a[order])))
    pct = samples / shape.n_total
    row = SweepRow("fps-b200", shape.dims[0], shape.dims[1] if shape.ndim > 1 else 1, k,
                   placement, trials, float(ok.mean()),
                   float(pct[ok].mean()) if ok.any() else math.nan, float(iters.mean()),
                   wall_ms)
    return row, dict(success=ok, samples_used=samples, iterations=iters,
                     terminated_by=res.terminated_by.cpu().numpy())


def run_sweep(shapes, k_values, placements, trials: int, seed: int,
              config: FpsSftConfig | None = None, **kw) -> list[SweepRow]:
    """Cells in the reference's order (``oracle.py:253-270``)."""
    config = config or FpsSftConfig(**PROFILES["P32"])
    rows = []
    for shape in shapes:
        shape = shape if isinstance(shape, CubeShape) else CubeShape(shape)
        for k in k_values:
            for placement in placements:
                rows.append(run_cell(shape, k, placement, trials, seed, config, **kw)[0])
    return rows
