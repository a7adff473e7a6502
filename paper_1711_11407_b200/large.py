"""The recovery loop for problems whose recovered set or lines do not fit one
CTA's shared memory: the imaging duality path (the
512 x 576 frequency cube has L = lcm(512, 576) = 4608 and up to ~20k
recovered pixels, in float64).

The loop is the reference's (``driver.py:121-212``, restated step for step in
``oracle/fps_oracle.py:recover``), driven from the host one step per launch:

  gather the D+1 lines      fpssft_gather_lines   (lines.py:36-64)
  1/L DFT of each line      fpssft_dft_forward    (transform.py:17-22)
  peel the recovered set    fpssft_project_onto_bins, one call per offset,
                            global-memory kernel for large sets
                            (decoder.py:172-191, driver.py:150-154)
  classify + decode + guard fpssft_decode_spectra (decoder.py:127-169,
                            driver.py:156-176)
  merge / prune / amp_sum   vectorised host slot arrays with the reference's
                            dict semantics and order (driver.py:94-118)
  peel the new entries,     device projection + max|S| (driver.py:189-204)
  termination

Default: the whole loop is one CUDA graph launch on the device
(``fpssft_recover_large``, csrc/fpssft_loop.cuh: a conditional WHILE node;
merge, amp_sum, residual and termination on the device, one host wait).
``loop="host"`` keeps the round-1 host-driven path (device steps, numpy merge)
for A/B.  There is no CPU fallback.
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from . import ops
from .core import CubeShape, SparseSpectrum
from .driver import (TERMINATED_MAX_ITERATIONS, TERMINATED_RESIDUAL_CLEAN, TERMINATED_STALL, _params,
                     C_ref, FpsSftConfig, IterationStats, RecoveryReport, _precision_code,
                     default_max_iterations)
from .schedule import schedule_from_seed


def stepped_offsets(tau, dims):
    """tau, tau + e_0, ..., tau + e_{D-1} (mod N_k) -- lines.py:55-64."""
    out = [tuple(int(v) for v in tau)]
    for k in range(len(dims)):
        t = list(out[0])
        t[k] = (t[k] + 1) % dims[k]
        out.append(tuple(t))
    return out


def line_spectra_global(cube, shape: CubeShape, alpha, tau, *, precision: str = "fp64"):
    """[D+1, L] spectra of one iteration's lines of one cube (complex64 or
    complex128 CUDA tensor), lines staged in global memory."""
    import torch

    D, L = shape.ndim, shape.line_len
    cube_prec = N.F64 if cube.dtype == torch.complex128 else N.F32
    if cube.dtype not in (torch.complex64, torch.complex128):
        raise TypeError("cube must be complex64 or complex128")
    at = torch.as_tensor(np.stack([np.asarray(alpha, np.int32), np.asarray(tau, np.int32)])[None],
                         device=cube.device)
    dt = torch.complex128 if _precision_code(precision) == N.F64 else torch.complex64
    lines = torch.empty((1, D + 1, L), dtype=dt, device=cube.device)
    sh = N.make_shape(shape.dims, [int(s) for s in cube.stride()])
    N.check(N.lib().fpssft_gather_lines(N.ptr(cube), cube_prec, 1, 0, C_ref(sh), N.ptr(at), 0,
                                        N.ptr(lines), _precision_code(precision),
                                        N.stream_ptr(cube.device)))
    return ops.dft_forward(lines, precision=precision)[0]


class _RecoveredSet:
    """The reference's recovered-set dict (driver.py:94-118) as slot arrays:
    slots in insertion order, a pruned key's slot zeroed and its key free to
    be re-appended at the end -- the same order a Python dict gives, so the
    device projections sum in the reference's order (a zero amplitude adds
    +0.0, which changes no sum).  Linear-index -> slot table for O(1)
    vectorised lookups; device copies grown by doubling."""

    def __init__(self, shape: CubeShape, device):
        import torch

        self.shape, self.device = shape, device
        self.slot_of = np.full(shape.n_total, -1, np.int64)
        self.keys = np.zeros(0, np.int64)
        self.freqs = np.zeros((0, shape.ndim), np.int32)
        self.amps = np.zeros(0, np.complex128)
        self.cap = 0
        self.d_freqs = torch.zeros((1, 1, shape.ndim), dtype=torch.int32, device=device)
        self.d_amps = torch.zeros((1, 1), dtype=torch.complex128, device=device)
        self.d_count = torch.zeros(1, dtype=torch.int32, device=device)
        self.n_up = 0

    def __len__(self):
        return int(np.count_nonzero(self.slot_of[self.keys] == np.arange(len(self.keys))))

    def merge(self, freqs: np.ndarray, amps: np.ndarray, prune_tol: float):
        """merge-by-sum then prune, for keys distinct within the call."""
        lin = np.ravel_multi_index(tuple(freqs.T), self.shape.dims)
        slot = self.slot_of[lin]
        old = slot >= 0
        v = self.amps[slot[old]] + amps[old]
        self.amps[slot[old]] = v
        dead = np.abs(v) <= prune_tol
        self.amps[slot[old][dead]] = 0j
        self.slot_of[lin[old][dead]] = -1
        fresh = ~old & ~(np.abs(0j + amps) <= prune_tol)
        n0 = len(self.keys)
        nf = int(np.count_nonzero(fresh))
        self.keys = np.concatenate([self.keys, lin[fresh]])
        self.freqs = np.concatenate([self.freqs, freqs[fresh].astype(np.int32)])
        self.amps = np.concatenate([self.amps, 0j + amps[fresh]])
        self.slot_of[lin[fresh]] = np.arange(n0, n0 + nf)

    def amp_total(self) -> float:
        live = self.slot_of[self.keys] == np.arange(len(self.keys))
        a = np.abs(self.amps[live])
        return float(np.cumsum(a)[-1]) if a.size else 0.0  # sequential, like sum()

    def upload(self):
        """Device copies (count = slots incl. zeroed ones)."""
        import torch

        n = len(self.keys)
        if n > self.cap:
            self.cap = max(n, 2 * self.cap, 64)
            f = torch.zeros((1, self.cap, self.shape.ndim), dtype=torch.int32, device=self.device)
            f[0, :self.n_up] = self.d_freqs[0, :self.n_up]
            self.d_freqs = f
            self.d_amps = torch.zeros((1, self.cap), dtype=torch.complex128, device=self.device)
        if n > self.n_up:
            self.d_freqs[0, self.n_up:n] = torch.as_tensor(self.freqs[self.n_up:n],
                                                           device=self.device)
            self.n_up = n
        self.d_amps[0, :n] = torch.as_tensor(self.amps, device=self.device)
        self.d_count.fill_(n)

    def entries(self):
        live = self.slot_of[self.keys] == np.arange(len(self.keys))
        return self.freqs[live].astype(np.int64), self.amps[live]


def _project(shape, freqs, amps, count, k_cap, at, out, precision, device, shape_c=None):
    """Device projection of (freqs, amps)[:count] onto the line whose
    (alpha, offset) int32 [1, 2, D] device tensor is ``at``, into ``out`` [1, L]
    (buffers made once per iteration by the caller: the loop is launch-bound)."""
    N.check(N.lib().fpssft_project_onto_bins(N.ptr(freqs), N.ptr(amps), N.ptr(count), 1, k_cap,
                                             C_ref(shape_c or N.make_shape(shape.dims)), N.ptr(at),
                                             0, N.ptr(out), _precision_code(precision),
                                             N.stream_ptr(device)))
    return out[0]


def fps_sft_large(cube, shape: CubeShape | None = None, config: FpsSftConfig = FpsSftConfig(),
                  *, precision: str = "fp64", schedule=None, loop: str = "device",
                  k_cap: int | None = None) -> RecoveryReport:
    """``fps_sft`` for a single large problem (CUDA tensor ``cube``).  Same
    arguments, defaults, schedule and report as the reference's entry point;
    float64 by default (the imaging path compares pixels to 1e-6).

    ``loop="device"`` (default, float64): the whole loop is one CUDA graph
    launch (``fpssft_recover_large``: a conditional WHILE node, the device
    decides termination, one host wait); ``loop="host"``: the host drives one
    device step per launch (the round-1 path, kept for A/B)."""
    if loop == "device" and _precision_code(precision) == N.F64:
        return _fps_sft_large_device(cube, shape, config, schedule, k_cap)
    if loop not in ("device", "host"):
        raise ValueError('loop must be "device" or "host"')
    return _fps_sft_large_host(cube, shape, config, precision=precision, schedule=schedule)


_RUNNERS: dict = {}  # persistent device buffers of the device loop, by shape


def _fps_sft_large_device(cube, shape, config, schedule, k_cap):
    """The device-resident loop (csrc/fpssft_loop.cuh)."""
    import torch

    shape = shape or CubeShape(tuple(cube.shape))
    if tuple(cube.shape) != shape.dims:
        raise ValueError(f"cube extents {tuple(cube.shape)} do not match {shape.dims}")
    if cube.dtype not in (torch.complex64, torch.complex128):
        raise TypeError("cube must be complex64 or complex128")
    if not cube.is_cuda:
        raise ValueError("cube must be a CUDA tensor")
    D, L = shape.ndim, shape.line_len
    dev = cube.device
    t_max = config.max_iterations or default_max_iterations(shape)
    if schedule is None:
        schedule = schedule_from_seed(shape, config.seed, t_max)
    schedule = np.ascontiguousarray(np.asarray(schedule, np.int32)[:t_max])
    if schedule.shape != (t_max, 2, D):
        raise ValueError(f"schedule must be [{t_max}, 2, {D}]")
    if k_cap is None:  # every slot a key may take, incl. re-appends after pruning
        k_cap = 1 << int(2 * shape.n_total - 1).bit_length()
    # persistent buffers per (device, shape, dtype, k_cap, t_max): the cube and
    # schedule are copied into them, so every pointer the library's graph bakes
    # in is stable and a repeated call only re-launches the cached graph
    rk = (str(dev), shape.dims, cube.dtype, k_cap, t_max)
    r = _RUNNERS.get(rk)
    lib = N.lib()
    if r is None:
        sh = N.make_shape(shape.dims)
        ws_bytes = int(lib.fpssft_recover_large_workspace(C_ref(sh), k_cap))
        if ws_bytes < 0:
            N.check(-1)
        r = dict(sh=sh, ws_bytes=ws_bytes,
                 ws=torch.empty(ws_bytes, dtype=torch.uint8, device=dev),
                 cube=torch.empty(shape.dims, dtype=cube.dtype, device=dev),
                 sched=torch.empty((t_max, 2, D), dtype=torch.int32, device=dev),
                 freqs=torch.empty((k_cap, D), dtype=torch.int32, device=dev),
                 amps=torch.empty(k_cap, dtype=torch.complex128, device=dev),
                 scal=torch.zeros(3, dtype=torch.int32, device=dev),  # count, iterations, term
                 samples=torch.zeros(1, dtype=torch.int64, device=dev),
                 stats=torch.zeros((t_max, 3), dtype=torch.int32, device=dev))
        if len(_RUNNERS) >= 4:
            _RUNNERS.pop(next(iter(_RUNNERS)))
        _RUNNERS[rk] = r
    r["cube"].copy_(cube)
    r["sched"].copy_(torch.as_tensor(schedule))
    params = _params(config, t_max, k_cap, N.F64)
    cube_prec = N.F64 if cube.dtype == torch.complex128 else N.F32
    scal, samples, stats, freqs, amps = r["scal"], r["samples"], r["stats"], r["freqs"], r["amps"]
    N.check(lib.fpssft_recover_large(N.ptr(r["cube"]), cube_prec, C_ref(r["sh"]), C_ref(params),
                                     N.ptr(r["sched"]), N.ptr(r["ws"]), r["ws_bytes"],
                                     N.ptr(freqs), N.ptr(amps), N.ptr(scal), N.ptr(scal[1:]),
                                     N.ptr(samples), N.ptr(scal[2:]), N.ptr(stats),
                                     N.stream_ptr(dev)))
    count, its, term = (int(v) for v in scal.cpu())
    f = freqs[:count].cpu().numpy().astype(np.int64)
    a = amps[:count].cpu().numpy()
    st = stats[:its].cpu().numpy()
    log = tuple(IterationStats(t + 1, tuple(int(v) for v in schedule[t, 0]),
                               tuple(int(v) for v in schedule[t, 1]), int(st[t, 0]),
                               int(st[t, 1]), int(st[t, 2])) for t in range(its))
    order = np.lexsort(f.T[::-1]) if count else np.zeros(0, np.int64)
    return RecoveryReport(iterations_run=its, samples_used=int(samples.item()),
                          recovered=SparseSpectrum._trusted(shape, f[order], a[order]),
                          terminated_by=N.TERM_NAMES[term], iteration_log=log)


def _fps_sft_large_host(cube, shape: CubeShape | None = None,
                        config: FpsSftConfig = FpsSftConfig(), *, precision: str = "fp64",
                        schedule=None) -> RecoveryReport:
    """Host-driven loop over device steps (one launch per step)."""
    import torch

    shape = shape or CubeShape(tuple(cube.shape))
    if tuple(cube.shape) != shape.dims:
        raise ValueError(f"cube extents {tuple(cube.shape)} do not match {shape.dims}")
    D, L, dims = shape.ndim, shape.line_len, shape.dims
    dev = cube.device
    t_max = config.max_iterations or default_max_iterations(shape)
    if schedule is None:
        schedule = schedule_from_seed(shape, config.seed, t_max)
    schedule = np.asarray(schedule)
    rs = _RecoveredSet(shape, dev)
    shape_c = N.make_shape(shape.dims)
    amp_total = 0.0
    stall, term, it = 0, TERMINATED_MAX_ITERATIONS, 0
    log = []
    for it in range(1, t_max + 1):
        alpha = tuple(int(v) for v in schedule[it - 1, 0])
        tau = tuple(int(v) for v in schedule[it - 1, 1])
        offs = stepped_offsets(tau, dims)
        spec = line_spectra_global(cube, shape, alpha, tau, precision=precision)
        spec = spec.to(torch.complex128)
        # the D+1 lines' (alpha, offset) and projection outputs, one transfer per iteration
        at_all = torch.as_tensor(np.stack([np.stack([np.asarray(alpha, np.int32),
                                                     np.asarray(off, np.int32)]) for off in offs]),
                                 device=dev)
        proj = torch.empty((D + 1, 1, L), dtype=torch.complex128, device=dev)
        if len(rs.keys):
            rs.upload()
            for i in range(D + 1):
                spec[i] -= _project(shape, rs.d_freqs, rs.d_amps, rs.d_count, rs.cap,
                                    at_all[i:i + 1], proj[i], precision, dev, shape_c)
        floor = max(config.energy_floor_abs, config.energy_floor * amp_total)
        st, fr, am, nc = ops.decode_spectra_device(spec[None], alpha, tau, shape, config, floor,
                                                   precision=precision)
        acc_t = torch.nonzero(st[0] == 2).flatten()  # ascending bins, guard applied
        new_f = fr[0, acc_t].cpu().numpy().astype(np.int64)
        new_a = am[0, acc_t].cpu().numpy()
        n_acc = len(new_a)
        if n_acc:  # merge-by-sum and prune (driver.py:103-108)
            rs.merge(new_f, new_a, config.amp_prune_tol)
        amp_total = rs.amp_total()
        n_cand = int(nc[0])
        log.append(IterationStats(it, alpha, tau, n_cand, n_acc, n_cand - n_acc))
        if n_acc:
            stall = 0
            nf = fr[0, acc_t].contiguous()[None]
            na = am[0, acc_t].contiguous()[None]
            cnt = torch.full((1,), n_acc, dtype=torch.int32, device=dev)
            for i in range(D + 1):
                spec[i] -= _project(shape, nf, na, cnt, n_acc, at_all[i:i + 1], proj[i],
                                    precision, dev, shape_c)
        else:
            stall += 1
        if float(spec.abs().max()) <= max(config.energy_floor_abs,
                                          config.residual_stop * amp_total):
            term = TERMINATED_RESIDUAL_CLEAN
            break
        if stall >= config.stall_limit:
            term = TERMINATED_STALL
            break
    freqs, amps = rs.entries()
    order = np.lexsort(freqs.T[::-1]) if len(freqs) else np.zeros(0, np.int64)
    return RecoveryReport(iterations_run=it, samples_used=it * (D + 1) * L,
                          recovered=SparseSpectrum._trusted(shape, freqs[order], amps[order]),
                          terminated_by=term, iteration_log=tuple(log))
