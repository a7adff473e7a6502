"""``baseline_sft`` on the GPU: the row/column comparison algorithm of the
paper (reference ``pkg/src/fps_sft/driver.py:219-314``).

Columns 0 and 1 and rows 0 and 1 are transformed once on the device
(``fpssft_line_spectra`` with slopes (1,0) and (0,1)); each iteration then
decodes one axis pass against the residual of those two spectra (projection
``fpssft_project_onto_bins``, classifier ``fpssft_decode_spectra`` on a 1-D
axis shape, no bin guard -- as the reference), and merges on the host.  It
is a comparison algorithm, not a throughput path: one pass per launch set.
"""

from __future__ import annotations

import numpy as np

from . import ops
from .core import CubeShape, SparseSpectrum
from .driver import (TERMINATED_MAX_ITERATIONS, TERMINATED_RESIDUAL_CLEAN, TERMINATED_STALL,
                     FpsSftConfig, IterationStats, RecoveryReport, default_max_iterations,
                     materialize)


def baseline_sft(source, config: FpsSftConfig = FpsSftConfig(), *, precision: str = "fp32",
                 device=None) -> RecoveryReport:
    import torch

    shape, cube = materialize(source, device)
    if shape.ndim != 2:
        raise ValueError("baseline recovery is defined for 2-D data only")
    n0, n1 = shape.dims
    if n0 != n1 or n0 < 1 or n0 & (n0 - 1):
        raise ValueError(f"baseline recovery requires equal power-of-two extents, got {shape.dims}")
    dev = torch.device(device if device is not None else "cuda")
    t = (cube if isinstance(cube, torch.Tensor) else torch.as_tensor(np.asarray(cube)))
    t = t.to(device=dev, dtype=torch.complex64).reshape(1, n0, n1)
    L = n0
    # line_spectra returns offsets tau, tau+e0, tau+e1: with slope (1,0) and
    # tau=(0,0) those are column 0 (twice, shifted) and column 1; with slope
    # (0,1), row 0 and row 1 (driver.py:238-245)
    cols = ops.line_spectra(t, (1, 0), (0, 0), precision=precision)[0]
    rows = ops.line_spectra(t, (0, 1), (0, 0), precision=precision)[0]
    base = {0: torch.stack([cols[0], cols[2]]).to(torch.complex128),
            1: torch.stack([rows[0], rows[1]]).to(torch.complex128)}
    passes = {0: ((1, 0), [(0, 0), (0, 1)], lambda b, m: (b, m)),
              1: ((0, 1), [(0, 0), (1, 0)], lambda b, m: (m, b))}
    axis = CubeShape([L])
    t_max = config.max_iterations or default_max_iterations(shape)
    entries: dict = {}
    amp_sum = 0.0
    log, stall, term, iterations = [], 0, TERMINATED_MAX_ITERATIONS, 0

    def residuals(ax):
        alpha, taus, _ = passes[ax]
        f = np.asarray(list(entries.keys()), np.int64).reshape(-1, 2)
        a = np.asarray(list(entries.values()), np.complex128)
        out = base[ax].clone()
        if len(a):
            for i, tau in enumerate(taus):
                out[i] -= ops.project_onto_bins(f, a, alpha, tau, shape, precision=precision,
                                                device=dev)
        return out

    for it in range(1, t_max + 1):
        iterations = it
        ax = (it - 1) % 2
        alpha, _, to_freq = passes[ax]
        spectra = residuals(ax)
        floor = max(config.energy_floor_abs, config.energy_floor * amp_sum)
        if precision == "fp32":
            # the float32 rounding floor of the fused loop is
            # set by the raw line energy, not by the (small) residual
            energy = L * float((base[ax].abs() ** 2).sum())  # sum |x|^2 (Parseval)
            floor = max(floor, 8 * 2.0**-24 * np.sqrt(np.log2(L) + 1) * np.sqrt(energy / 2) / L)
        st, fr, am, nc = ops.decode_spectra_device(spectra[None], (1,), (0,), axis, config, floor,
                                                   precision=precision)
        st, fr, am = st[0].cpu().numpy(), fr[0].cpu().numpy(), am[0].cpu().numpy()
        accepted = [(to_freq(int(b), int(fr[b, 0])), complex(am[b]))
                    for b in np.flatnonzero(st >= 2)]  # decoder semantics: no bin guard
        for f, a in accepted:  # merge-by-sum and prune (driver.py:103-108)
            v = entries.get(f, 0j) + a
            entries[f] = v
            if abs(v) <= config.amp_prune_tol:
                del entries[f]
        amp_sum = sum(abs(v) for v in entries.values())
        n_cand = int(nc[0])
        log.append(IterationStats(it, alpha, (0, 0), n_cand, len(accepted),
                                  n_cand - len(accepted)))
        stall = 0 if accepted else stall + 1
        clean = max(config.energy_floor_abs, config.residual_stop * amp_sum)
        worst = max(float(residuals(0).abs().max()), float(residuals(1).abs().max()))
        if worst <= clean:
            term = TERMINATED_RESIDUAL_CLEAN
            break
        if stall >= config.stall_limit:
            term = TERMINATED_STALL
            break
    return RecoveryReport(iterations_run=iterations, samples_used=4 * L,
                          recovered=SparseSpectrum(shape, entries), terminated_by=term,
                          iteration_log=tuple(log))
