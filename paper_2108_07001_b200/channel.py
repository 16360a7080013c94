"""Fiber channel on the GPU: float64 FFTs of any length and the split-step
Fourier span (the step before the receive path).

`fft` / `ifft` are numpy.fft.fft / ifft over the last axis (kk_fft: Stockham
passes for powers of two, Bluestein's chirp-z otherwise).  `ssfm_span` is
kkmodem's channel.ssfm_span (channel.py:124-158) with the same arguments,
parameter derivation, errors and return type, and its FFT / dispersion /
nonlinear-phase steps in kk_ssfm_span -- the nonlinear link of acceptance C8
(test_acceptance.py:268-320) runs through it when the kkmodem backend switch
is installed (kkmodem_backend.py).  Results equal the reference to float64
rounding (tests/test_gpu_channel.py), not bit for bit: pocketfft and this
FFT order their butterflies differently.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .sigcore import ParameterError, cd_phase_coefficient


def _torch():
    import torch
    return torch


def _as_device_c128(x, device=None):
    torch = _torch()
    if isinstance(x, torch.Tensor):
        t = x.to(torch.complex128)
        if not t.is_cuda:
            t = t.to(device or torch.device("cuda", torch.cuda.current_device()))
        return t.contiguous(), True
    arr = np.ascontiguousarray(np.asarray(x, dtype=np.complex128))
    dev = device or torch.device("cuda", torch.cuda.current_device())
    return torch.from_numpy(arr).to(dev), False


def _transform(x, inverse: bool):
    torch = _torch()
    t, was_torch = _as_device_c128(x)
    n = int(t.shape[-1]) if t.dim() else 0
    if n == 0:
        raise ParameterError("fft of an empty sequence")
    batch = int(t.numel() // n)
    nws = int(_lib.load().kk_fft_workspace_bytes(n, batch))
    if nws == 0:
        raise ParameterError("fft length too large")
    ws = torch.empty(nws, dtype=torch.uint8, device=t.device)
    out = torch.empty_like(t)
    _lib.call("kk_fft", t.data_ptr(), out.data_ptr(), n, batch, int(inverse), ws.data_ptr(), nws,
              torch.cuda.current_stream(t.device).cuda_stream)
    return out if was_torch else out.cpu().numpy()


def fft(x):
    """numpy.fft.fft over the last axis, float64, on the GPU (numpy in ->
    numpy out; a torch tensor in -> a CUDA complex128 tensor out)."""
    return _transform(x, False)


def ifft(x):
    """numpy.fft.ifft over the last axis (1/n normalisation), on the GPU."""
    return _transform(x, True)


def ssfm_span(signal, span, step_km: float | None = None, lambda_nm: float = 1550.116):
    """Propagate one span with the symmetric split-step Fourier method
    (channel.py ssfm_span :124-158): per step half-step dispersion, the
    nonlinear phase rotation over the step's effective length, half-step
    dispersion, then the step's loss.  `signal`: any object with .samples
    (numpy or torch complex) and .sample_rate_hz; returns an object of the
    same type (kkmodem's ComplexSignal under the switch)."""
    torch = _torch()
    if step_km is None:
        step_km = 1.0
    if step_km <= 0:
        raise ParameterError("step_km must be positive")
    step_km = min(step_km, span.length_km) if span.length_km > 0 else step_km
    n_steps = max(1, int(round(span.length_km / step_km)))
    dz = span.length_km / n_steps
    alpha = span.loss_db_per_km * np.log(10.0) / 10.0
    a_half = cd_phase_coefficient(span.dispersion_ps_nm_km, dz / 2.0, lambda_nm)
    l_eff = (1.0 - np.exp(-alpha * dz)) / alpha if alpha > 0 else dz
    loss_amp = np.exp(-alpha * dz / 2.0)
    fs = float(signal.sample_rate_hz)
    x, was_torch = _as_device_c128(signal.samples)
    x = x.clone() if was_torch else x          # the caller's tensor is not modified
    n = int(x.shape[0])
    nws = int(_lib.load().kk_ssfm_workspace_bytes(n))
    if nws == 0:
        raise ParameterError("signal too long for the split-step span")
    ws = torch.empty(nws, dtype=torch.uint8, device=x.device)
    _lib.call("kk_ssfm_span", x.data_ptr(), n, fs, n_steps, float(a_half), float(span.gamma_per_w_km),
              float(l_eff), float(loss_amp), ws.data_ptr(), nws, torch.cuda.current_stream(x.device).cuda_stream)
    out = x if was_torch else x.cpu().numpy()
    return type(signal)(out, signal.sample_rate_hz)
