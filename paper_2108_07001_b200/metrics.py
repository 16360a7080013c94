"""Link metrics on decided streams (kkmodem.metrics, metrics.py:69-179).

BER counting over long streams runs on the GPU (`count_bit_errors`, the
kk_bit_errors kernel = demap + XOR popcount of runner.py:360-362, with the
windowed counts of metrics.py:133-151).  The scalar formulas (Q from BER,
EVM) and the bit-level frame_sync used by the small-capture `measure_point`
are host-side arithmetic, restated from the reference.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .constellation import slicer_tables
from .sigcore import ParameterError


class SyncFailure(RuntimeError):
    """Bit streams could not be aligned (metrics.py:27)."""


def q_from_ber(ber: float) -> float:
    """20 log10(sqrt(2) erfcinv(2 BER)) (metrics.py:121-130)."""
    from scipy.special import erfcinv

    if ber == 0:
        return float("inf")
    if not (0.0 < ber < 0.5):
        raise ParameterError("ber must be in (0, 0.5)")
    return float(20.0 * np.log10(np.sqrt(2.0) * erfcinv(2.0 * ber)))


def evm(soft_symbols, reference_symbols) -> float:
    """RMS error over RMS reference, percent (metrics.py:170-179)."""
    s, r = np.asarray(soft_symbols), np.asarray(reference_symbols)
    if len(s) != len(r):
        raise ParameterError("sequences must have equal length")
    if len(r) == 0:
        raise ParameterError("sequences are empty")
    return float(100.0 * np.sqrt(np.mean(np.abs(s - r) ** 2) / np.mean(np.abs(r) ** 2)))


def frame_sync(rx_bits, tx_bits, min_peak_ratio: float = 3.0):
    """Bipolar cross-correlation alignment (metrics.py:69-112)."""
    from scipy.signal import fftconvolve

    rx = np.asarray(rx_bits, dtype=np.int8) * 2 - 1
    tx = np.asarray(tx_bits, dtype=np.int8) * 2 - 1
    if len(tx) < (1 << 14):
        raise ParameterError("reference must be at least 2^14 bits")
    if len(rx) < 64:
        raise SyncFailure("received stream too short")
    if len(rx) == len(tx):
        c = np.fft.ifft(np.fft.fft(rx) * np.conj(np.fft.fft(tx))).real
        mag = np.abs(c)
        k = int(np.argmax(mag))
        ratio = mag[k] / (np.max(np.delete(mag, k)) + 1e-30)
        if ratio < min_peak_ratio:
            raise SyncFailure(f"no circular correlation peak (ratio {ratio:.2f})")
        return k, np.roll(np.asarray(rx_bits, dtype=np.uint8), -k), np.asarray(tx_bits, dtype=np.uint8)
    c = fftconvolve(rx.astype(np.float64), tx[::-1].astype(np.float64), mode="full")
    mag = np.abs(c)
    k = int(np.argmax(mag))
    side = np.delete(mag, np.arange(max(0, k - 2), min(len(mag), k + 3)))
    ratio = mag[k] / (np.max(side) + 1e-30)
    if ratio < min_peak_ratio:
        raise SyncFailure(f"no correlation peak (ratio {ratio:.2f})")
    lag = (len(tx) - 1) - k
    ru, tu = np.asarray(rx_bits, dtype=np.uint8), np.asarray(tx_bits, dtype=np.uint8)
    if lag >= 0:
        n = min(len(ru), len(tu) - lag)
        return lag, ru[:n], tu[lag:lag + n]
    n = min(len(ru) + lag, len(tu))
    return lag, ru[-lag:-lag + n], tu[:n]


def windowed_q(error_flags, bit_rate_hz: float, window_s: float = 0.021):
    """Per-window Q with the one-error floor (metrics.py:133-151)."""
    flags = np.asarray(error_flags)
    bpw = int(round(window_s * bit_rate_hz))
    if bpw < 1 or len(flags) < bpw:
        raise ParameterError("stream shorter than one window")
    n_win = len(flags) // bpw
    return [(k * window_s, q_from_ber(max(int(np.sum(flags[k * bpw:(k + 1) * bpw])), 1) / bpw))
            for k in range(n_win)]


def windowed_q_from_counts(counts, bits_per_window: int, window_s: float):
    """windowed_q from per-window error counts produced on the GPU."""
    return [(k * window_s, q_from_ber(max(int(c), 1) / bits_per_window)) for k, c in enumerate(counts)]


def count_bit_errors(labels, ref_idx, order: int, window_symbols: int = 0, exclude_period: int = 0,
                     exclude_len: int = 0, exclude_phase: int = 0):
    """GPU bit-error count between decided point indices and transmitted
    point indices (both uint8 CUDA tensors of equal length).  Symbols i with
    (i + exclude_phase) % exclude_period >= exclude_period - exclude_len are
    skipped (tile seams).  Returns device tensors (errors[1], symbols[1]) and
    the per-window counts (or None)."""
    import torch

    n = int(labels.shape[0])
    if int(ref_idx.shape[0]) != n:
        raise ParameterError("labels and reference must have equal length")
    tb = slicer_tables(order)
    dev = labels.device
    from .rxdsp import _device_const

    pl = _device_const("point_label", tb.point_label, dev)   # no per-call upload
    tot = torch.zeros(1, dtype=torch.int64, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    win = None
    if window_symbols > 0:
        win = torch.zeros(max(1, -(-n // window_symbols)), dtype=torch.int32, device=dev)
    _lib.call("kk_bit_errors", labels.data_ptr(), ref_idx.data_ptr(), n, pl.data_ptr(), int(window_symbols),
              tot.data_ptr(), win.data_ptr() if win is not None else None, int(exclude_period),
              int(exclude_len), int(exclude_phase), cnt.data_ptr(), torch.cuda.current_stream(dev).cuda_stream)
    return tot, cnt, win
