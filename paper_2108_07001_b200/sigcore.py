"""Host-side signal containers and plan/constant helpers.

Mirrors the parts of kkmodem.sigcore the receiver API exposes
(sigcore.py:37-147 types, :217-230 `fir_frequency_response`, :302-316
`anti_alias_window`, :170-214 `design_rrc`, :357-398 raw int16/f32 I/O).
These are setup-time constants (filter responses, plans), evaluated once per
pipeline in float64 on the host exactly as the reference does; the per-sample
work all runs in the CUDA library.

Signal containers additionally accept torch CUDA tensors so device-resident
streams never round-trip through host memory.
"""

from __future__ import annotations

import importlib
import importlib.util
import json
import os
import sys
from dataclasses import dataclass, field

import numpy as np


def kkmodem_class(module: str, name: str):
    """kkmodem's own class `module.name` when the reference package is
    importable (so errors raised here are caught by the reference's callers,
    e.g. runner.py:182 `except (SyncError, SyncFailure)`), else None.
    The repo-local reference install (baseline/_ref, tools/install_reference.py)
    is used when kkmodem is not otherwise importable.  KKB200_NO_KKMODEM=1
    disables the lookup."""
    if os.environ.get("KKB200_NO_KKMODEM") == "1":
        return None
    try:
        if importlib.util.find_spec("kkmodem") is None:
            ref = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
            if not os.path.isdir(os.path.join(ref, "kkmodem")):
                return None
            os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/kkb200_numba_cache")
            sys.path.append(ref)
        return getattr(importlib.import_module(module), name)
    except Exception:   # a broken or partial kkmodem install: stand alone
        return None


_KK_PARAMETER_ERROR = kkmodem_class("kkmodem.sigcore", "ParameterError")


class ParameterError(*((_KK_PARAMETER_ERROR,) if _KK_PARAMETER_ERROR else (ValueError,))):
    """Raised when an operation receives arguments violating its contract
    (kkmodem.sigcore.ParameterError, sigcore.py:37; a subclass of it when
    kkmodem is importable)."""


def is_signal(x) -> bool:
    """Duck-typed signal container (this package's or kkmodem's
    RealSignal/ComplexSignal, sigcore.py:46-99): has .samples and
    .sample_rate_hz."""
    return hasattr(x, "samples") and hasattr(x, "sample_rate_hz")


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


@dataclass
class ComplexSignal:
    """Uniformly sampled complex waveform (sigcore.py:46-82).  `samples` is
    a numpy complex128 array or a torch complex tensor (device resident)."""

    samples: object
    sample_rate_hz: float

    def __post_init__(self):
        if not _is_torch(self.samples):
            self.samples = np.asarray(self.samples, dtype=np.complex128)
        if self.sample_rate_hz <= 0:
            raise ParameterError("sample_rate_hz must be positive")

    def __len__(self) -> int:
        return int(self.samples.shape[0])


@dataclass
class RealSignal:
    """Uniformly sampled real waveform (sigcore.py:85-99)."""

    samples: object
    sample_rate_hz: float

    def __post_init__(self):
        if not _is_torch(self.samples):
            self.samples = np.asarray(self.samples, dtype=np.float64)
        if self.sample_rate_hz <= 0:
            raise ParameterError("sample_rate_hz must be positive")

    def __len__(self) -> int:
        return int(self.samples.shape[0])


@dataclass
class AdcCodes:
    """Exact ADC wire format: odd half-LSB int16 codes h with value
    h * half_lsb (the mid-rise levels (code + 0.5) * lsb of frontend.py:108-117;
    the int16 raw format of sigcore.py:357-377).  numpy int16 or a torch
    int16 tensor."""

    codes: object
    half_lsb: float
    sample_rate_hz: float = 4e9

    def __len__(self) -> int:
        return int(self.codes.shape[0])

    def to_real(self) -> RealSignal:
        return RealSignal(np.asarray(self.codes, dtype=np.float64) * self.half_lsb, self.sample_rate_hz)


@dataclass
class AdcPacked12:
    """Packed 12-bit wire format (B200 addition; 1.5 B/sample): the 12-bit
    ADC codes c (frontend.py:82-118, h = 2c + 1 the odd half-LSB code of
    AdcCodes, value h * half_lsb) two per 3 bytes, little-endian (byte0 =
    c0[7:0], byte1 = c0[11:8] | c1[3:0] << 4, byte2 = c1[11:4]).  `data`:
    uint8 numpy array or torch tensor of >= 3 n / 2 bytes; n even."""

    data: object
    half_lsb: float
    n: int
    sample_rate_hz: float = 4e9

    def __post_init__(self):
        if self.n % 2:
            raise ParameterError("packed 12-bit streams hold an even number of samples")
        if int(self.data.shape[0]) < 3 * self.n // 2:
            raise ParameterError("packed buffer shorter than 3 n / 2 bytes")

    def __len__(self) -> int:
        return int(self.n)


def pack12(codes_h) -> np.ndarray:
    """int16 odd half-LSB codes h = 2c + 1 (|c| < 2048) -> packed 12-bit bytes."""
    h = np.asarray(codes_h, dtype=np.int32)
    if len(h) % 2:
        raise ParameterError("packed 12-bit streams hold an even number of samples")
    if np.any((h & 1) == 0) or np.any(h < -4095) or np.any(h > 4095):
        raise ParameterError("codes must be odd half-LSB codes of a 12-bit converter")
    c = ((h - 1) >> 1) & 0xFFF
    c0, c1 = c[0::2], c[1::2]
    out = np.empty((len(h) // 2, 3), dtype=np.uint8)
    out[:, 0] = c0 & 0xFF
    out[:, 1] = (c0 >> 8) | ((c1 & 0xF) << 4)
    out[:, 2] = c1 >> 4
    return out.reshape(-1)


def unpack12(data, n: int) -> np.ndarray:
    """Packed 12-bit bytes -> int16 odd half-LSB codes (host reference of
    kk_unpack12)."""
    b = np.asarray(data, dtype=np.uint8)[:3 * n // 2].reshape(-1, 3).astype(np.int32)
    c0 = b[:, 0] | ((b[:, 1] & 0xF) << 8)
    c1 = (b[:, 1] >> 4) | (b[:, 2] << 4)
    c = np.empty(n, dtype=np.int32)
    c[0::2], c[1::2] = c0, c1
    c = (c ^ 0x800) - 0x800
    return (2 * c + 1).astype(np.int16)


@dataclass
class FirFilter:
    """FIR taps with the rate they are defined at (sigcore.py:102-118)."""

    taps: np.ndarray
    nominal_rate_hz: float

    def __post_init__(self):
        self.taps = np.asarray(self.taps, dtype=np.complex128)
        if len(self.taps) < 1:
            raise ParameterError("filter needs at least one tap")
        if self.nominal_rate_hz <= 0:
            raise ParameterError("nominal_rate_hz must be positive")
        if not np.all(np.isfinite(self.taps)):
            raise ParameterError("taps contains non-finite samples")

    def __len__(self) -> int:
        return len(self.taps)


@dataclass
class BlockPlan:
    """100 % overlap-save plan: hop == fft_size/2 (sigcore.py:121-147)."""

    fft_size: int = 1024
    hop: int = field(default=0)
    buffer_len: int = 1 << 22

    def __post_init__(self):
        n = self.fft_size
        if n < 2 or (n & (n - 1)) != 0:
            raise ParameterError("fft_size must be a power of two >= 2")
        if self.hop == 0:
            self.hop = n // 2
        if self.hop != n // 2:
            raise ParameterError("hop must equal fft_size/2")
        if self.buffer_len % self.hop != 0:
            raise ParameterError("buffer_len must be a multiple of hop")

    @property
    def blocks_per_buffer(self) -> int:
        return self.buffer_len // self.hop


def fir_frequency_response(fir, freqs_hz, rate_hz: float | None = None) -> np.ndarray:
    """DTFT of causal taps at the given frequencies (sigcore.py:217-230)."""
    if hasattr(fir, "taps") and hasattr(fir, "nominal_rate_hz"):   # this package's or kkmodem's FirFilter
        taps, rate = fir.taps, (fir.nominal_rate_hz if rate_hz is None else rate_hz)
    else:
        if rate_hz is None:
            raise ParameterError("rate_hz required for bare tap arrays")
        taps, rate = np.asarray(fir, dtype=np.complex128), rate_hz
    f = np.asarray(freqs_hz, dtype=np.float64)
    return np.exp(-2j * np.pi * np.outer(f, np.arange(len(taps))) / rate) @ taps


def anti_alias_window(freqs_hz, nyquist_hz: float, edge: float = 0.01) -> np.ndarray:
    """Brick wall with a raised-cosine edge (sigcore.py:302-316)."""
    a = np.abs(np.asarray(freqs_hz, dtype=np.float64))
    f_pass = nyquist_hz * (1.0 - edge)
    w = np.where(a <= f_pass, 1.0, 0.0)
    t = (a > f_pass) & (a < nyquist_hz)
    w[t] = 0.5 * (1.0 + np.cos(np.pi * (a[t] - f_pass) / (nyquist_hz - f_pass)))
    return w


def design_rrc(rolloff: float, sps: int, span_symbols: int) -> FirFilter:
    """Unit-energy root-raised-cosine (sigcore.py:170-214); used by the
    host-side receive-tap design only."""
    if not (0.0 < rolloff <= 1.0):
        raise ParameterError("rolloff must be in (0, 1]")
    if sps < 2:
        raise ParameterError("sps must be >= 2")
    if span_symbols < 2 or span_symbols % 2:
        raise ParameterError("span_symbols must be an even integer >= 2")
    n = span_symbols * sps
    t = (np.arange(n + 1) - n / 2) / sps
    b = rolloff
    h = np.empty(n + 1)
    at = np.abs(t)
    zero = at < 1e-12
    sing = np.abs(at - 1.0 / (4.0 * b)) < 1e-9
    reg = ~(zero | sing)
    tr = t[reg]
    h[reg] = (np.sin(np.pi * tr * (1 - b)) + 4 * b * tr * np.cos(np.pi * tr * (1 + b))) / (
        np.pi * tr * (1 - (4 * b * tr) ** 2))
    h[zero] = 1.0 - b + 4.0 * b / np.pi
    h[sing] = (b / np.sqrt(2.0)) * ((1 + 2 / np.pi) * np.sin(np.pi / (4 * b))
                                    + (1 - 2 / np.pi) * np.cos(np.pi / (4 * b)))
    h /= np.sqrt(np.sum(h * h))
    return FirFilter(h, float(sps))


def cd_phase_coefficient(dispersion_ps_nm_km: float, length_km: float, lambda_nm: float) -> float:
    """a in H(f) = exp(-j a f^2) (channel.py:82-87)."""
    c = 299792458.0
    return np.pi * (dispersion_ps_nm_km * 1e-6) * (lambda_nm * 1e-9) ** 2 * (length_km * 1e3) / c


def write_adc_raw(path: str, adc: AdcCodes) -> None:
    """int16 raw + JSON sidecar (the wire format of sigcore.py:357-382,
    storing the exact odd half-LSB codes: value = code / scale)."""
    np.asarray(adc.codes, dtype="<i2").tofile(path)
    with open(path + ".json", "w") as f:
        json.dump({"sample_rate_hz": adc.sample_rate_hz, "length": len(adc), "kind": "int16",
                   "scale": 1.0 / adc.half_lsb}, f, sort_keys=True)


def read_adc_raw(path: str) -> AdcCodes:
    """Read an int16 raw stream (sigcore.py:385-398) without converting to
    float: value = code / scale."""
    with open(path + ".json") as f:
        meta = json.load(f)
    if meta["kind"] != "int16":
        raise ParameterError("not an int16 raw stream")
    return AdcCodes(np.fromfile(path, dtype="<i2"), 1.0 / meta["scale"], meta["sample_rate_hz"])
