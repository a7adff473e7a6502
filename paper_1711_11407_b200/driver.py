"""The FPS-SFT entry points: ``fps_sft`` (drop-in for the reference's) and
``fps_sft_batch`` (many independent instances per launch).

Mirrors ``fps_sft.driver`` (``/root/reference/pkg/src/fps_sft/driver.py``):
``FpsSftConfig`` (:29-63, same fields, defaults and validation),
``IterationStats`` (:66-73), ``RecoveryReport`` (:76-85),
``default_max_iterations`` (:88-91) and ``fps_sft(source, config)``
(:121-212).  The loop itself runs on the GPU in one fused kernel per batch
(``csrc/fpssft.cu:recover_kernel``) reached through the C ABI
``fpssft_run_batch``; this module only prepares the schedule, owns the
buffers and unpacks results.  Without a CUDA device or the built library it
raises -- there is no CPU path.

Deliberate differences:
* The schedule (alpha_t, tau_t) is explicit.  ``fps_sft`` derives it from
  ``config.seed`` exactly as the reference draws it (``schedule.py``), so the
  same seed follows the same lines.
* Arithmetic is float32 (the north-star configuration): plain
  (``precision="fp32"``) for tight noiseless profiles, guarded
  (``"fp32-guarded"``: float64 amplitudes, every decision inside its float32
  error bound of the threshold re-evaluated in float64) for the loose noisy
  profiles -- ``"auto"`` (default) picks by the profile; ``"fp64"`` runs the
  kernels in float64.
* ``time_domain_subtraction`` is accepted for signature compatibility; the
  device path always subtracts in the frequency domain (the reference states
  both give identical results up to roundoff, driver.py:37-41).
* The recovered set has a capacity ``k_cap``; exceeding it ends that
  instance with ``terminated_by == "k_cap_overflow"`` (never silently).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .core import CubeShape, DenseSource, SignalSource, SparseSpectrum
from .schedule import schedule_from_seed

TERMINATED_RESIDUAL_CLEAN = "residual_clean"
TERMINATED_STALL = "stall"
TERMINATED_MAX_ITERATIONS = "max_iterations"
TERMINATED_K_CAP_OVERFLOW = "k_cap_overflow"

DEFAULT_MAG_TOL = 1e-6
DEFAULT_VERIFY_TOL = 1e-6
DEFAULT_ROUND_TOL = 0.05
DEFAULT_AMP_PRUNE_TOL = 1e-9
DEFAULT_ENERGY_FLOOR_REL = 1e-9
DEFAULT_ENERGY_FLOOR_ABS = 1e-12


@dataclass(frozen=True)
class FpsSftConfig:
    max_iterations: int | None = None
    stall_limit: int = 3
    seed: int = 0
    mag_tol: float = DEFAULT_MAG_TOL
    verify_tol: float = DEFAULT_VERIFY_TOL
    round_tol: float = DEFAULT_ROUND_TOL
    amp_prune_tol: float = DEFAULT_AMP_PRUNE_TOL
    energy_floor: float = DEFAULT_ENERGY_FLOOR_REL
    energy_floor_abs: float = DEFAULT_ENERGY_FLOOR_ABS
    residual_stop: float = 1e-9
    time_domain_subtraction: bool = False

    def __post_init__(self):
        if self.max_iterations is not None and self.max_iterations < 1:
            raise ValueError("max_iterations must be >= 1")
        if self.stall_limit < 1:
            raise ValueError("stall_limit must be >= 1")
        for name in ("mag_tol", "verify_tol", "round_tol", "amp_prune_tol",
                     "energy_floor", "energy_floor_abs", "residual_stop"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive")


# Tolerance profiles used by the configs.
PROFILES = {
    "P64": {},
    "P32": dict(mag_tol=1e-4, verify_tol=1e-4, residual_stop=1e-6),
    "PN": dict(mag_tol=0.3, verify_tol=0.5, round_tol=0.3),
}


@dataclass(frozen=True)
class IterationStats:
    iteration: int
    alpha: tuple[int, ...]
    tau: tuple[int, ...]
    candidates: int
    accepted: int
    rejected: int


@dataclass(frozen=True)
class RecoveryReport:
    iterations_run: int
    samples_used: int
    recovered: SparseSpectrum
    terminated_by: str
    iteration_log: tuple[IterationStats, ...] = field(default=())

    def percent_samples(self) -> float:
        return self.samples_used / self.recovered.shape.n_total


def default_max_iterations(shape: CubeShape) -> int:
    return max(1, shape.n_total // ((shape.ndim + 1) * shape.line_len))


def _precision_code(precision: str, config=None) -> int:
    """``fp32`` | ``fp64`` | ``fp32-guarded`` (float32 arithmetic with the
    float64 reference's decisions, csrc/fpssft_guard.cuh) | ``auto``:
    guarded for loose (noisy-data) tolerance profiles, where decision
    statistics land near their thresholds, plain float32 otherwise."""
    if precision == "auto":
        loose = config is not None and max(config.mag_tol, config.verify_tol) >= 1e-3
        return N.F32_GUARDED if loose else N.F32
    if precision in ("fp32", "float32", "f32"):
        return N.F32
    if precision in ("fp64", "float64", "f64"):
        return N.F64
    if precision in ("fp32-guarded", "fp32g", "guarded"):
        return N.F32_GUARDED
    raise ValueError(f"unknown precision {precision!r}")


def _params(config: FpsSftConfig, t_max: int, k_cap: int, precision: int,
            mode: str = "auto") -> N.Params:
    p = N.Params()
    p.t_max, p.stall_limit, p.k_cap, p.precision = t_max, config.stall_limit, k_cap, precision
    if mode not in N.MODES:
        raise ValueError(f"mode must be one of {sorted(N.MODES)}")
    p.mode = N.MODES[mode]
    for name in ("mag_tol", "verify_tol", "round_tol", "amp_prune_tol", "energy_floor",
                 "energy_floor_abs", "residual_stop"):
        setattr(p, name, float(getattr(config, name)))
    return p


def C_ref(x):
    import ctypes

    return ctypes.byref(x)


def _pow2_ceil(x: int) -> int:
    return 1 << max(0, int(x - 1).bit_length())


def max_k_cap(shape: CubeShape, precision: str = "fp32", mode: str = "auto",
              config=None) -> int:
    """Largest power-of-two capacity whose on-chip state fits (in ``mode``)."""
    sh = N.make_shape(shape.dims)
    best = 0
    k = 1
    while k <= (1 << 20):
        p = _params(FpsSftConfig(), 1, k, _precision_code(precision, config), mode)
        if N.lib().fpssft_smem_bytes(C_ref(sh), C_ref(p)) == 0:  # no plan fits
            break
        best = k
        k <<= 1
    return best


@dataclass
class BatchResult:
    """Padded per-instance outputs of one ``fps_sft_batch`` call (device tensors)."""

    shape: CubeShape
    k_cap: int
    freqs: "object"  # int32 [B, k_cap, D]
    amps: "object"  # complex128 [B, k_cap]
    count: "object"  # int32 [B]
    iterations: "object"  # int32 [B]
    samples_used: "object"  # int64 [B]
    terminated_by: "object"  # int32 [B]
    iter_stats: "object" = None  # int32 [B, t_max, 3] or None
    schedule: np.ndarray | None = None  # int32 [S, t_max, 2, D] (host copy)
    sched_index: np.ndarray | None = None

    @property
    def batch(self) -> int:
        return int(self.count.shape[0])

    def report(self, b: int) -> RecoveryReport:
        """The reference-shaped report of instance ``b`` (host copy)."""
        n = int(self.count[b])
        freqs = self.freqs[b, :n].cpu().numpy().astype(np.int64)
        amps = self.amps[b, :n].cpu().numpy()
        its = int(self.iterations[b])
        term = N.TERM_NAMES[int(self.terminated_by[b])]
        log = ()
        if self.iter_stats is not None and self.schedule is not None:
            s = 0 if self.sched_index is None else int(self.sched_index[b])
            st = self.iter_stats[b, :its].cpu().numpy()
            sch = self.schedule[s]
            log = tuple(IterationStats(t + 1, tuple(int(v) for v in sch[t, 0]),
                                       tuple(int(v) for v in sch[t, 1]), int(st[t, 0]),
                                       int(st[t, 1]), int(st[t, 2])) for t in range(its))
        return RecoveryReport(iterations_run=its, samples_used=int(self.samples_used[b]),
                              recovered=SparseSpectrum._trusted(self.shape, freqs, amps),
                              terminated_by=term, iteration_log=log)


class Outputs(dict):
    """The per-instance output tensors, all views of one allocation ``buf``
    (so a whole batch's results move host<->device in one copy)."""

    buf: "object" = None


_OUT_FIELDS = (("freqs", "int32", 4), ("amps", "complex128", 16), ("count", "int32", 4),
               ("iterations", "int32", 4), ("samples_used", "int64", 8),
               ("terminated_by", "int32", 4), ("iter_stats", "int32", 4))


def allocate_outputs(batch: int, shape: CubeShape, k_cap: int, t_max: int, device,
                     iter_stats: bool = False, pin: bool = False) -> Outputs:
    """Zeroed output tensors for ``batch`` instances, packed in one buffer
    (pinned host memory with ``pin``)."""
    import torch

    shapes = {"freqs": (batch, k_cap, shape.ndim), "amps": (batch, k_cap), "count": (batch,),
              "iterations": (batch,), "samples_used": (batch,), "terminated_by": (batch,),
              "iter_stats": (batch, t_max, 3) if iter_stats else None}
    offs, o = {}, 0
    for name, _, size in _OUT_FIELDS:
        if shapes[name] is None:
            continue
        o = (o + 15) // 16 * 16
        offs[name] = o
        n = 1
        for d in shapes[name]:
            n *= d
        o += n * size
    buf = torch.zeros(max(16, o), dtype=torch.uint8, device=device, pin_memory=pin)
    out = Outputs()
    for name, dt, size in _OUT_FIELDS:
        if shapes[name] is None:
            out[name] = None
            continue
        n = 1
        for d in shapes[name]:
            n *= d
        out[name] = buf[offs[name]:offs[name] + n * size].view(getattr(torch, dt)).view(
            shapes[name])
    out.buf = buf
    return out


def _schedule_tensor(schedule, shape: CubeShape, t_max: int, device):
    import torch

    sch = np.asarray(schedule, dtype=np.int32)
    if sch.ndim == 3:
        sch = sch[None]
    if sch.ndim != 4 or sch.shape[2:] != (2, shape.ndim):
        raise ValueError(f"schedule must be [S, T, 2, {shape.ndim}], got {sch.shape}")
    if sch.shape[1] < t_max:
        raise ValueError(f"schedule holds {sch.shape[1]} iterations, t_max is {t_max}")
    sch = np.ascontiguousarray(sch[:, :t_max])
    dims = np.asarray(shape.dims)
    if (sch < 0).any() or (sch >= dims).any():
        raise ValueError("schedule slope/offset components out of range")
    return sch, torch.as_tensor(sch, device=device)


class BatchRunner:
    """Pre-planned launcher for repeated batches of one shape: schedule on the
    device, outputs allocated once, one ``fpssft_run_batch`` per ``run``."""

    def __init__(self, shape: CubeShape, config: FpsSftConfig, batch: int, *, schedule=None,
                 sched_index=None, k_cap: int = 256, precision: str = "auto",
                 iter_stats: bool = False, device=None, mode: str = "auto", group: int = 1,
                 stage_iterations: int = 0):
        import torch

        if not 1 <= int(group) <= 64:
            raise ValueError("group must be in [1, 64]")
        self.group = int(group)
        # stage_iterations > 0 (interleaved batch, one schedule): the line
        # samples of the first iterations are staged through HBM by TMA bulk
        # copies (``fpssft_run_batch_staged``: a pinned host batch then crosses
        # the link at its bulk rate instead of the SM loads' request rate)
        self.stage_iterations = int(stage_iterations)
        if self.stage_iterations < 0:
            raise ValueError("stage_iterations must be >= 0")
        if self.stage_iterations and (self.group < 2 or self.group % 2 or sched_index is not None):
            raise ValueError("staged lines need an interleaved batch (even group) that shares "
                             "one schedule")
        self.shape = shape
        self.config = config
        self.batch = int(batch)
        self.device = torch.device(device if device is not None else "cuda")
        self.t_max = config.max_iterations or default_max_iterations(shape)
        if schedule is None:
            schedule = schedule_from_seed(shape, config.seed, self.t_max)
        self.schedule_host, self.schedule = _schedule_tensor(schedule, shape, self.t_max,
                                                             self.device)
        self.sched_index_host = None
        self.sched_index = None
        if sched_index is not None:
            si = np.asarray(sched_index, dtype=np.int32).reshape(-1)
            if si.shape[0] != self.batch:
                raise ValueError("sched_index must have one entry per instance")
            if (si < 0).any() or (si >= self.schedule_host.shape[0]).any():
                raise ValueError("sched_index out of range")
            self.sched_index_host = si
            self.sched_index = torch.as_tensor(si, device=self.device)
        if k_cap < 1 or k_cap & (k_cap - 1):
            raise ValueError("k_cap must be a positive power of two")
        self.k_cap = int(k_cap)
        self.prec = _precision_code(precision, config)
        self._shape_c = N.make_shape(shape.dims)
        self._params_c = _params(config, self.t_max, self.k_cap, self.prec, mode)
        self.plan = launch_plan(shape, self._params_c, self.group, self.sched_index is not None)
        self.out = allocate_outputs(self.batch, shape, self.k_cap, self.t_max, self.device,
                                    iter_stats)
        o = self.out
        self._out_c = N.Out(N.ptr(o["freqs"]), N.ptr(o["amps"]), N.ptr(o["count"]),
                            N.ptr(o["iterations"]), N.ptr(o["samples_used"]),
                            N.ptr(o["terminated_by"]), N.ptr(o["iter_stats"]))
        self.smem_bytes = self.plan["smem_bytes"]
        self.threads = self.plan["threads_per_cta"]
        self._staging = None
        if self.stage_iterations:
            if self.schedule_host.shape[0] != 1:
                raise ValueError("staged lines need a single schedule")
            nbytes = int(N.lib().fpssft_stage_bytes(C_ref(self._shape_c), self.group, self.batch,
                                                    min(self.stage_iterations, self.t_max)))
            if nbytes < 0:
                raise ValueError("staged lines: unsupported shape / group")
            self._staging = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=self.device)

    def _check_cubes(self, cubes):
        import torch

        if not isinstance(cubes, torch.Tensor):
            raise ValueError("cubes must be a CUDA tensor (use fps_sft for host arrays)")
        if not cubes.is_cuda and not cubes.is_pinned():
            raise ValueError("cubes must be a CUDA tensor or a pinned host tensor "
                             "(use fps_sft for other host arrays)")
        if cubes.dtype != torch.complex64:
            raise ValueError(f"cubes must be complex64, got {cubes.dtype}")
        G = self.group
        if G == 1:
            if tuple(cubes.shape[1:]) != self.shape.dims or cubes.shape[0] != self.batch:
                raise ValueError(f"cubes must be [{self.batch}, {self.shape.dims}], "
                                 f"got {tuple(cubes.shape)}")
            strides = [int(s) for s in cubes.stride()[1:]]
        else:  # interleaved batch [ceil(B/G), *dims, G] (see ``interleave``)
            want = ((self.batch + G - 1) // G, *self.shape.dims, G)
            if tuple(cubes.shape) != want or cubes.stride(-1) != 1:
                raise ValueError(f"grouped cubes must be {want} with unit last stride, "
                                 f"got {tuple(cubes.shape)}")
            strides = [int(s) for s in cubes.stride()[1:-1]]
        # element strides (complex64 units) of one cube and between cubes (groups)
        return N.make_shape(self.shape.dims, strides)

    def stage(self, cubes) -> None:
        """The staging pass alone (``stage_iterations`` > 0), on the current
        stream; ``run(cubes, staged=True)`` then skips it."""
        if self._staging is None:
            raise ValueError("this runner was built without stage_iterations")
        sh = self._check_cubes(cubes)
        dev = cubes.device if cubes.is_cuda else self.device
        import torch

        with torch.cuda.device(dev):
            N.check(N.lib().fpssft_stage_lines(
                N.ptr(cubes), self.batch, self.group, int(cubes.stride(0)), C_ref(sh),
                C_ref(self._params_c), N.ptr(self.schedule), N.ptr(self._staging),
                int(self._staging.numel()), self.stage_iterations, N.stream_ptr(dev)))

    def run(self, cubes, staged: bool = False) -> BatchResult:
        import torch

        sh = self._check_cubes(cubes)
        G = self.group
        # a pinned host tensor is read in place by the kernel (zero copy over the
        # host link: only the gathered samples cross it, the sub-linear sample
        # budget of the algorithm); its UVA address is valid on the device
        dev = cubes.device if cubes.is_cuda else self.device
        with torch.cuda.device(dev):
            if self._staging is not None:
                N.check(N.lib().fpssft_run_batch_staged(
                    N.ptr(cubes), self.batch, G, int(cubes.stride(0)), C_ref(sh),
                    C_ref(self._params_c), N.ptr(self.schedule), C_ref(self._out_c),
                    N.ptr(self._staging), int(self._staging.numel()), self.stage_iterations,
                    int(bool(staged)), N.stream_ptr(dev)))
            else:
                N.check(N.lib().fpssft_run_batch_grouped(
                    N.ptr(cubes), self.batch, G, int(cubes.stride(0)), C_ref(sh),
                    C_ref(self._params_c), N.ptr(self.schedule), N.ptr(self.sched_index),
                    int(self.schedule_host.shape[0]), C_ref(self._out_c), N.stream_ptr(dev)))
        o = self.out
        return BatchResult(self.shape, self.k_cap, o["freqs"], o["amps"], o["count"],
                           o["iterations"], o["samples_used"], o["terminated_by"],
                           o["iter_stats"], self.schedule_host, self.sched_index_host)


def interleave(cubes, group: int = 8):
    """The interleaved batch layout ``[ceil(B/G), *dims, G]`` of ``[B, *dims]``
    cubes (a copy; the last group zero-padded): sample n of G consecutive
    instances shares one 64-byte DRAM segment at G = 8, so a schedule shared
    by the batch reads every segment once for G instances instead of once per
    instance.  Run it with ``BatchRunner(..., group=G)``."""
    import torch

    B, dims = int(cubes.shape[0]), tuple(cubes.shape[1:])
    ng = (B + group - 1) // group
    out = torch.zeros((ng, *dims, group), dtype=cubes.dtype, device=cubes.device)
    full = B // group
    nd = len(dims)
    if full:
        out[:full].copy_(cubes[:full * group].reshape(full, group, *dims)
                         .permute(0, *range(2, nd + 2), 1))
    for b in range(full * group, B):
        out[full][..., b - full * group] = cubes[b]
    return out


def launch_plan(shape: CubeShape, params: N.Params, group: int = 1,
                per_instance_schedules: bool = False) -> dict:
    """The kernel/launch shape ``fpssft_run_batch_grouped`` will use for a
    batch interleaved by ``group`` (raises if the shape cannot run)."""
    import ctypes

    mode, thr, per = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    smem = ctypes.c_size_t()
    N.check(N.lib().fpssft_plan_batch(C_ref(N.make_shape(shape.dims)), C_ref(params), int(group),
                                      int(bool(per_instance_schedules)), C_ref(mode), C_ref(thr),
                                      C_ref(per), C_ref(smem)))
    return {"mode": {N.MODE_CTA: "cta", N.MODE_WARP: "warp"}[mode.value],
            "threads_per_cta": thr.value, "instances_per_cta": per.value,
            "smem_bytes": smem.value}


def fps_sft_batch(cubes, config: FpsSftConfig = FpsSftConfig(), *, schedule=None,
                  sched_index=None, k_cap: int = 256, precision: str = "auto",
                  iter_stats: bool = False, mode: str = "auto") -> BatchResult:
    """Recover every instance of ``cubes`` (complex64 CUDA tensor [B, *dims]).

    ``schedule``: int32 [T, 2, D] or [S, T, 2, D] (alpha, tau) per iteration;
    default: the reference's draws for ``config.seed``.  ``sched_index``:
    per-instance schedule row (default 0).  Returns padded device tensors.
    """
    shape = CubeShape(cubes.shape[1:])
    runner = BatchRunner(shape, config, cubes.shape[0], schedule=schedule,
                         sched_index=sched_index, k_cap=k_cap, precision=precision,
                         iter_stats=iter_stats, device=cubes.device, mode=mode)
    return runner.run(cubes)


def materialize(source, device=None) -> tuple[CubeShape, "np.ndarray | object"]:
    """The dense complex64 cube behind a sample source: a ``DenseSource``'s
    own array; for a lazy sinusoid mixture that exposes its spectrum (the
    reference's ``SyntheticSource.spectrum``, core.py:176-217) the grid is
    synthesised on the device (``fpssft_synthesize``);
    otherwise ``sample_many`` over the whole grid on the host."""
    shape = source.shape()
    if not isinstance(shape, CubeShape):
        shape = CubeShape(shape.dims)
    if isinstance(source, DenseSource):
        return shape, source.data
    data = getattr(source, "_data", None)  # the reference's DenseSource
    if isinstance(data, np.ndarray) and data.shape == shape.dims:
        return shape, data.astype(np.complex64)
    spec = getattr(source, "spectrum", None)
    if spec is not None and hasattr(spec, "freq_array") and hasattr(spec, "amp_array"):
        import torch

        from .ops import synthesize

        f = np.asarray(spec.freq_array, np.int32).reshape(-1, shape.ndim)
        a = np.asarray(spec.amp_array, np.complex128)
        k = max(1, len(a))
        kc = 1 << (k - 1).bit_length()
        fr = np.zeros((1, kc, shape.ndim), np.int32)
        am = np.zeros((1, kc), np.complex128)
        fr[0, :len(a)], am[0, :len(a)] = f, a
        dev = torch.device(device if device is not None else "cuda")
        cube = synthesize(torch.as_tensor(fr, device=dev), torch.as_tensor(am, device=dev),
                          torch.as_tensor(np.asarray([len(a)], np.int32), device=dev),
                          shape=shape, precision="fp64")
        return shape, cube[0]
    if shape.n_total > (1 << 24):
        raise ValueError(f"refusing to materialise a lazy source of {shape.n_total} samples")
    grid = np.indices(shape.dims).reshape(shape.ndim, -1).T
    return shape, source.sample_many(grid).reshape(shape.dims).astype(np.complex64)


def fps_sft(source: SignalSource, config: FpsSftConfig = FpsSftConfig(), *,
            precision: str = "auto", k_cap: int | None = None, device=None,
            mode: str = "auto") -> RecoveryReport:
    """Recover the sparse spectrum of ``source`` on the GPU (driver.py:121-212).

    Same contract as the reference: stops on a clean residual, after
    ``stall_limit`` fruitless iterations, or at the iteration cap; failure to
    recover is reported, never raised.
    """
    import torch

    shape, cube = materialize(source, device)
    dev = torch.device(device if device is not None else "cuda")
    if isinstance(cube, torch.Tensor):
        t = cube.to(device=dev, dtype=torch.complex64)
    else:
        t = torch.as_tensor(np.ascontiguousarray(cube, dtype=np.complex64)).to(dev)
    t = t.reshape((1, *shape.dims))
    if k_cap is None:
        k_cap = min(_pow2_ceil(shape.n_total), max_k_cap(shape, precision, mode, config))
        if k_cap < 1:
            raise N.UnsupportedError(f"shape {shape.dims} does not fit one CTA")
    res = fps_sft_batch(t, config, k_cap=k_cap, precision=precision, iter_stats=True, mode=mode)
    return res.report(0)


__all__ = ["FpsSftConfig", "IterationStats", "RecoveryReport", "BatchResult", "BatchRunner",
           "default_max_iterations", "fps_sft", "fps_sft_batch", "launch_plan", "materialize",
           "max_k_cap",
           "PROFILES", "TERMINATED_RESIDUAL_CLEAN", "TERMINATED_STALL",
           "TERMINATED_MAX_ITERATIONS", "TERMINATED_K_CAP_OVERFLOW"]
