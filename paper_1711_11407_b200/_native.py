"""ctypes binding of the C ABI in ``include/fpssft.h`` (libfpssft.so).

There is no fallback: if the shared library is missing or a call fails, the
caller gets an exception.  Device buffers are passed as raw pointers of CUDA
tensors; the stream is the caller's current torch stream.
"""

from __future__ import annotations

import ctypes as C
import os

LIB_PATH = os.environ.get("FPSSFT_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "libfpssft.so")  # FPSSFT_LIB: A/B builds
MAX_DIMS = 4

F32, F64, F32_GUARDED = 0, 1, 2
MODE_AUTO, MODE_CTA, MODE_WARP = 0, 1, 2
MODES = {"auto": MODE_AUTO, "cta": MODE_CTA, "warp": MODE_WARP}
TERM_NAMES = {0: "residual_clean", 1: "stall", 2: "max_iterations", 3: "k_cap_overflow",
              -1: "invalid_schedule"}

EXPORTS = ("fpssft_run_batch", "fpssft_run_batch_grouped", "fpssft_run_batch_staged",
           "fpssft_stage_bytes", "fpssft_stage_lines", "fpssft_line_spectra", "fpssft_gather_lines", "fpssft_dft_forward",
           "fpssft_synthesize", "fpssft_recover_large", "fpssft_recover_large_workspace",
           "fpssft_decode_spectra", "fpssft_project_onto_bins", "fpssft_smem_bytes",
           "fpssft_block_threads", "fpssft_plan", "fpssft_plan_batch", "fpssft_launches_per_batch",
           "fpssft_set_l2_fetch_granularity", "fpssft_get_l2_fetch_granularity", "fpssft_last_error",
           "fpssft_abi_version")


class Shape(C.Structure):
    _fields_ = [("ndim", C.c_int32), ("dims", C.c_int32 * MAX_DIMS),
                ("strides", C.c_int64 * MAX_DIMS)]


class Params(C.Structure):
    _fields_ = [("t_max", C.c_int32), ("stall_limit", C.c_int32), ("k_cap", C.c_int32),
                ("precision", C.c_int32), ("mode", C.c_int32), ("mag_tol", C.c_double), ("verify_tol", C.c_double),
                ("round_tol", C.c_double), ("amp_prune_tol", C.c_double),
                ("energy_floor", C.c_double), ("energy_floor_abs", C.c_double),
                ("residual_stop", C.c_double)]


class Out(C.Structure):
    _fields_ = [("freqs", C.c_void_p), ("amps", C.c_void_p), ("count", C.c_void_p),
                ("iterations", C.c_void_p), ("samples_used", C.c_void_p),
                ("terminated_by", C.c_void_p), ("iter_stats", C.c_void_p)]


class FpsSftError(RuntimeError):
    pass


class UnsupportedError(ValueError):
    """Shape / capacity beyond what one CTA can hold on chip."""


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with "
                              "`python -c 'import __graft_entry__ as g; g.build()'`")
        h = C.CDLL(LIB_PATH)
        P, I32, I64 = C.c_void_p, C.c_int32, C.c_int64
        h.fpssft_run_batch.argtypes = [P, I64, I64, C.POINTER(Shape), C.POINTER(Params), P, P,
                                       I32, C.POINTER(Out), P]
        h.fpssft_run_batch_grouped.argtypes = [P, I64, I32, I64, C.POINTER(Shape),
                                               C.POINTER(Params), P, P, I32, C.POINTER(Out), P]
        h.fpssft_run_batch_staged.argtypes = [P, I64, I32, I64, C.POINTER(Shape),
                                              C.POINTER(Params), P, C.POINTER(Out), P, I64, I32,
                                              I32, P]
        h.fpssft_stage_lines.argtypes = [P, I64, I32, I64, C.POINTER(Shape), C.POINTER(Params),
                                         P, P, I64, I32, P]
        h.fpssft_stage_bytes.argtypes = [C.POINTER(Shape), I32, I64, I32]
        h.fpssft_stage_bytes.restype = I64
        h.fpssft_line_spectra.argtypes = [P, I64, I64, C.POINTER(Shape), P, I32, P, I32, P]
        h.fpssft_dft_forward.argtypes = [P, I64, I32, P, I32, P]
        h.fpssft_gather_lines.argtypes = [P, I32, I64, I64, C.POINTER(Shape), P, I32, P, I32, P]
        h.fpssft_decode_spectra.argtypes = [P, I64, C.POINTER(Shape), P, I32, C.POINTER(Params),
                                            C.c_double, P, P, P, P, P]
        h.fpssft_project_onto_bins.argtypes = [P, P, P, I64, I32, C.POINTER(Shape), P, I32, P,
                                               I32, P]
        h.fpssft_synthesize.argtypes = [P, P, P, I64, I32, C.POINTER(Shape), P, I64, I32, P]
        h.fpssft_recover_large_workspace.argtypes = [C.POINTER(Shape), I32]
        h.fpssft_recover_large_workspace.restype = I64
        h.fpssft_recover_large.argtypes = [P, I32, C.POINTER(Shape), C.POINTER(Params), P, P,
                                           I64, P, P, P, P, P, P, P, P]
        h.fpssft_smem_bytes.argtypes = [C.POINTER(Shape), C.POINTER(Params)]
        h.fpssft_smem_bytes.restype = C.c_size_t
        h.fpssft_block_threads.argtypes = [C.POINTER(Shape), I32]
        h.fpssft_plan.argtypes = [C.POINTER(Shape), C.POINTER(Params), C.POINTER(I32),
                                  C.POINTER(I32), C.POINTER(I32), C.POINTER(C.c_size_t)]
        h.fpssft_plan_batch.argtypes = [C.POINTER(Shape), C.POINTER(Params), I32, I32,
                                        C.POINTER(I32), C.POINTER(I32), C.POINTER(I32),
                                        C.POINTER(C.c_size_t)]
        h.fpssft_set_l2_fetch_granularity.argtypes = [I32]
        h.fpssft_get_l2_fetch_granularity.argtypes = []
        h.fpssft_last_error.restype = C.c_char_p
        for name in EXPORTS:
            if name not in ("fpssft_smem_bytes", "fpssft_last_error",
                            "fpssft_recover_large_workspace", "fpssft_stage_bytes"):
                getattr(h, name).restype = C.c_int
        _lib = h
    return _lib


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().fpssft_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise OverflowError(msg)
    if rc == 3:
        raise UnsupportedError(msg)
    raise FpsSftError(msg)


def make_shape(dims, strides=None) -> Shape:
    dims = [int(d) for d in dims]
    if not 1 <= len(dims) <= MAX_DIMS:
        raise UnsupportedError(f"the device path supports 1..{MAX_DIMS} dimensions, got {len(dims)}")
    if strides is None:
        strides, acc = [], 1
        for d in reversed(dims):
            strides.append(acc)
            acc *= d
        strides.reverse()
    s = Shape()
    s.ndim = len(dims)
    for k, (d, st) in enumerate(zip(dims, strides)):
        s.dims[k] = d
        s.strides[k] = int(st)
    return s


def ptr(t) -> int | None:
    return None if t is None else int(t.data_ptr())


def stream_ptr(device=None) -> int:
    import torch

    return int(torch.cuda.current_stream(device).cuda_stream)


def set_l2_fetch_granularity(nbytes: int, device=None) -> None:
    """cudaLimitMaxL2FetchGranularity for ``device`` (process-wide, opt-in)."""
    import torch

    with torch.cuda.device(device if device is not None else torch.cuda.current_device()):
        check(lib().fpssft_set_l2_fetch_granularity(int(nbytes)))


def get_l2_fetch_granularity(device=None) -> int:
    import torch

    with torch.cuda.device(device if device is not None else torch.cuda.current_device()):
        return int(lib().fpssft_get_l2_fetch_granularity())
