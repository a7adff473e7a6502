"""Device versions of the reference's per-step functions, for parity tests
and for callers that want one step at a time.  Each goes through the C ABI
and runs the same device code the fused loop uses.

=========================  ===============================================
here                       reference (``pkg/src/fps_sft/``)
=========================  ===============================================
``line_spectra``           [dft_forward(extract_line(DenseSource, (alpha,
                           off))) for off in decoding_offsets(tau)]
                           (lines.py:36-64, core.py:236-238, transform.py:17)
``dft_forward``            transform.py:17-22
``decode_spectra``         decoder.py:127-169 (+ driver.py:166-176 guard)
``project_onto_bins``      decoder.py:172-191
=========================  ===============================================
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from .core import CubeShape, Sinusoid
from .driver import C_ref, FpsSftConfig, _params, _precision_code


def _ctype(precision: str):
    import torch

    return torch.complex128 if _precision_code(precision) == N.F64 else torch.complex64


def _alpha_tau(alpha, tau, D, device):
    import torch

    at = np.stack([np.asarray(alpha, np.int32).reshape(-1, D),
                   np.asarray(tau, np.int32).reshape(-1, D)], axis=1)
    return torch.as_tensor(np.ascontiguousarray(at), device=device), int(at.shape[0] > 1)


def line_spectra(cubes, alpha, tau, *, precision: str = "fp32"):
    """[B, D+1, L] spectra of the D+1 lines of one iteration per cube.
    ``cubes``: complex64 CUDA tensor [B, *dims]; alpha/tau: (D,) or (B, D)."""
    import torch

    shape = CubeShape(cubes.shape[1:])
    D, L, B = shape.ndim, shape.line_len, cubes.shape[0]
    at, per = _alpha_tau(alpha, tau, D, cubes.device)
    out = torch.empty((B, D + 1, L), dtype=_ctype(precision), device=cubes.device)
    sh = N.make_shape(shape.dims, [int(s) for s in cubes.stride()[1:]])
    N.check(N.lib().fpssft_line_spectra(N.ptr(cubes), B, int(cubes.stride(0)), C_ref(sh),
                                        N.ptr(at), per, N.ptr(out), _precision_code(precision),
                                        N.stream_ptr(cubes.device)))
    return out


def dft_forward(lines, *, precision: str = "fp32"):
    """1/L-normalised forward DFT along the last axis of a CUDA tensor."""
    import torch

    if lines.ndim < 1 or lines.shape[-1] < 1:
        raise ValueError("expected a nonempty array")
    L = int(lines.shape[-1])
    x = lines.to(_ctype(precision)).contiguous()
    out = torch.empty_like(x)
    B = x.numel() // L
    N.check(N.lib().fpssft_dft_forward(N.ptr(x), B, L, N.ptr(out), _precision_code(precision),
                                       N.stream_ptr(x.device)))
    return out


def decode_spectra_device(spectra, alpha, tau, shape: CubeShape, config: FpsSftConfig,
                          floor: float, *, precision: str = "fp32"):
    """Raw classifier output per bin: (status [B, L], freqs [B, L, D],
    amps [B, L] complex128, n_candidates [B]).  status: 0 not a candidate,
    1 rejected, 2 accepted, 3 decoded but failed the bin guard."""
    import torch

    D, L = shape.ndim, shape.line_len
    sp = spectra.to(_ctype(precision)).contiguous().reshape(-1, D + 1, L)
    B = sp.shape[0]
    dev = sp.device
    at, per = _alpha_tau(alpha, tau, D, dev)
    status = torch.empty((B, L), dtype=torch.int32, device=dev)
    freqs = torch.empty((B, L, D), dtype=torch.int32, device=dev)
    amps = torch.empty((B, L), dtype=torch.complex128, device=dev)
    ncand = torch.empty(B, dtype=torch.int32, device=dev)
    p = _params(config, 1, 1, _precision_code(precision))
    N.check(N.lib().fpssft_decode_spectra(N.ptr(sp), B, C_ref(N.make_shape(shape.dims)),
                                          N.ptr(at), per, C_ref(p), float(floor), N.ptr(status),
                                          N.ptr(freqs), N.ptr(amps), N.ptr(ncand),
                                          N.stream_ptr(dev)))
    return status, freqs, amps, ncand


def decode_spectra(spectra, tau, shape: CubeShape, *, alpha=None, mag_tol=1e-6, round_tol=0.05,
                   verify_tol=1e-6, energy_floor=1e-12, precision: str = "fp32"):
    """Reference-shaped ``decode_spectra`` for one (D+1, L) spectra array:
    returns ([(bin, Sinusoid)] in ascending bin order, n_candidates).  Without
    ``alpha`` the bin guard is not applied (decoder.py semantics); with it,
    guard failures are dropped (the driver's filter)."""
    import torch

    cfg = FpsSftConfig(mag_tol=mag_tol, round_tol=round_tol, verify_tol=verify_tol)
    t = spectra if isinstance(spectra, torch.Tensor) else torch.as_tensor(np.asarray(spectra))
    if not t.is_cuda:
        t = t.cuda()
    al = alpha if alpha is not None else (1,) * shape.ndim
    st, fr, am, nc = decode_spectra_device(t, al, tau, shape, cfg, energy_floor,
                                           precision=precision)
    st, fr, am = st[0].cpu().numpy(), fr[0].cpu().numpy(), am[0].cpu().numpy()
    keep = st == 2 if alpha is not None else st >= 2
    out = [(int(b), Sinusoid(amp=complex(am[b]), freq=tuple(int(v) for v in fr[b])))
           for b in np.flatnonzero(keep)]
    return out, int(nc[0])


def project_onto_bins(freqs, amps, alpha, tau, shape: CubeShape, *, precision: str = "fp32",
                      device=None):
    """Length-L spectrum of a sparse set on the line (alpha, tau); sums in
    entry order (decoder.py:172-191).  Returns a complex128 CUDA tensor."""
    import torch

    dev = torch.device(device if device is not None else "cuda")
    f = np.asarray(freqs, np.int32).reshape(-1, shape.ndim)
    a = np.asarray(amps, np.complex128).reshape(-1)
    K = max(1, f.shape[0])
    kcap = 1 << max(0, int(K - 1).bit_length())
    fb = np.zeros((1, kcap, shape.ndim), np.int32)
    ab = np.zeros((1, kcap), np.complex128)
    fb[0, :f.shape[0]] = f
    ab[0, :a.shape[0]] = a
    ft = torch.as_tensor(fb, device=dev)
    atn = torch.as_tensor(ab, device=dev)
    cnt = torch.as_tensor(np.asarray([f.shape[0]], np.int32), device=dev)
    at, per = _alpha_tau(alpha, tau, shape.ndim, dev)
    out = torch.empty((1, shape.line_len), dtype=torch.complex128, device=dev)
    N.check(N.lib().fpssft_project_onto_bins(N.ptr(ft), N.ptr(atn), N.ptr(cnt), 1, kcap,
                                             C_ref(N.make_shape(shape.dims)), N.ptr(at), per,
                                             N.ptr(out), _precision_code(precision),
                                             N.stream_ptr(dev)))
    return out[0]


def synthesize(result_or_freqs, amps=None, counts=None, *, shape: CubeShape | None = None,
               precision: str = "fp32", out=None):
    """Dense complex64 grid of every instance's recovered spectrum
    (x(n) = sum_i a_i exp(+2 pi j sum_k n_k m_ik / N_k), the dense form of
    SyntheticSource.sample_many, core.py:176-217).  Accepts a ``BatchResult``
    or device tensors (freqs [B,k,D] int32, amps [B,k] complex128, counts [B])."""
    import torch

    if amps is None:
        res = result_or_freqs
        freqs, amps, counts, shape = res.freqs, res.amps, res.count, res.shape
    else:
        freqs = result_or_freqs
    B, k_cap = int(freqs.shape[0]), int(freqs.shape[1])
    dev = freqs.device
    if out is None:
        out = torch.empty((B, *shape.dims), dtype=torch.complex64, device=dev)
    elif not out.is_cuda and not out.is_pinned():
        # a pinned host ``out`` is written in place over the host link
        raise ValueError("out must be a CUDA tensor or a pinned host tensor")
    N.check(N.lib().fpssft_synthesize(N.ptr(freqs.contiguous()), N.ptr(amps.contiguous()),
                                      N.ptr(counts.contiguous()), B, k_cap,
                                      C_ref(N.make_shape(shape.dims)), N.ptr(out),
                                      int(out.stride(0)) if B else 0,
                                      _precision_code(precision), N.stream_ptr(dev)))
    return out
