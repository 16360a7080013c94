"""ORACLE -- TEST INFRASTRUCTURE ONLY.

CPU float64 restatement of the reference receiver hot path
(/root/reference/pkg/src/kkmodem/rxdsp.py, abbreviated `rx`; sigcore.py `sc`;
txdsp.py `tx`; metrics.py `me`; harness/runner.py `hr`).

Only tests/, `__graft_entry__.smoke()` and bench.py's `cpu_baseline` /
`--impl reference` legs may import this module, and only as the checker or
the timed CPU baseline -- never as the product.  The product
(`paper_2108_07001_b200`) never imports anything under oracle/ and fails
loudly when its CUDA library is missing.

Parity pinning: tests/test_oracle.py checks this restatement against the
golden fixtures in tests/golden/, which tools/gen_golden.py produced by
running the REAL reference (`RxPipeline` via `receive_stream`,
`measure_point`) in the build container.  The KK / carrier / downshift /
static stages reproduce the reference bit-for-bit (same numpy FFT calls, same
expression order); the DDLMS recurrence (oracle/ddlms_core.c, plain C with
-ffp-contract=off) reproduces the reference decisions exactly.

Arithmetic is numpy (pocketfft) + scipy.signal.fftconvolve, exactly the
third-party calls the reference makes.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np
from numpy.lib.stride_tricks import sliding_window_view

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


# ---------------------------------------------------------------------------
# constellations (tx:115-142); QPSK table tx:36-41, 8-QAM ring ratio tx:46,
# 32-cross labels tx:52-63, square Gray tx:102-112
# ---------------------------------------------------------------------------

_QPSK = {0: 1 + 1j, 1: -1 + 1j, 3: -1 - 1j, 2: 1 - 1j}
_CROSS32 = {
    (-5, -3): 25, (-5, -1): 29, (-5, 1): 31, (-5, 3): 27, (-3, -5): 26, (-3, -3): 24,
    (-3, -1): 13, (-3, 1): 15, (-3, 3): 11, (-3, 5): 9, (-1, -5): 30, (-1, -3): 28,
    (-1, -1): 12, (-1, 1): 14, (-1, 3): 10, (-1, 5): 8, (1, -5): 22, (1, -3): 20,
    (1, -1): 4, (1, 1): 6, (1, 3): 2, (1, 5): 0, (3, -5): 18, (3, -3): 16,
    (3, -1): 5, (3, 1): 7, (3, 3): 3, (3, 5): 1, (5, -3): 17, (5, -1): 21,
    (5, 1): 23, (5, 3): 19,
}


@dataclass
class Constellation:
    order: int
    points: np.ndarray
    labels: np.ndarray

    @property
    def bits_per_symbol(self) -> int:
        return int(np.log2(self.order))

    @property
    def max_radius(self) -> float:
        return float(np.max(np.abs(self.points)))


def constellation(order: int) -> Constellation:
    """Restates make_constellation (tx:115-142)."""
    if order == 4:
        labs = np.array(sorted(_QPSK))
        pts = np.array([_QPSK[k] for k in labs])
    elif order == 8:
        ratio = (1.0 + np.sqrt(3.0)) / np.sqrt(2.0)
        gray4 = [0, 1, 3, 2]
        pts, labs = [], []
        for ring, (rad, degs) in enumerate([(1.0, [45, 135, 225, 315]),
                                            (ratio, [0, 90, 180, 270])]):
            for q, a in enumerate(np.deg2rad(degs)):
                pts.append(rad * np.exp(1j * a))
                labs.append((ring << 2) | gray4[q])
        pts, labs = np.array(pts), np.array(labs)
    elif order in (16, 64):
        m = int(np.sqrt(order))
        lv = np.arange(-(m - 1), m, 2, dtype=np.float64)
        kb = int(np.log2(m))
        gray = [i ^ (i >> 1) for i in range(m)]
        pts = np.array([lv[a] + 1j * lv[b] for a in range(m) for b in range(m)])
        labs = np.array([(gray[a] << kb) | gray[b] for a in range(m) for b in range(m)])
    elif order == 32:
        items = sorted(_CROSS32.items())
        pts = np.array([i + 1j * q for (i, q), _ in items])
        labs = np.array([v for _, v in items])
    else:
        raise ValueError(order)
    pts = pts / np.sqrt(np.mean(np.abs(pts) ** 2))
    return Constellation(order, pts.astype(np.complex128), labs.astype(np.int64))


# ---------------------------------------------------------------------------
# static response (rx:401-411, sc:217-230, sc:302-316)
# ---------------------------------------------------------------------------

def fir_response(taps: np.ndarray, freqs: np.ndarray, rate: float) -> np.ndarray:
    m = np.arange(len(taps))
    return np.exp(-2j * np.pi * np.outer(freqs, m) / rate) @ taps


def aa_window(freqs: np.ndarray, nyq: float, edge: float) -> np.ndarray:
    a = np.abs(np.asarray(freqs, dtype=np.float64))
    fp = nyq * (1.0 - edge)
    w = np.zeros_like(a)
    w[a <= fp] = 1.0
    t = (a > fp) & (a < nyq)
    w[t] = 0.5 * (1.0 + np.cos(np.pi * (a[t] - fp) / (nyq - fp)))
    return w


def static_response(taps: np.ndarray, taps_rate: float, n: int, fs_in: float,
                    edge: float, aa_delay: int):
    m = n // 2
    kept = np.concatenate([np.arange(0, m // 2), np.arange(n - m // 2, n)])
    f = np.fft.fftfreq(n, 1.0 / fs_in)[kept]
    h = fir_response(np.asarray(taps, np.complex128), f, taps_rate)
    h *= aa_window(f, fs_in / 4.0, edge)
    h *= np.exp(-2j * np.pi * f * aa_delay / fs_in)
    return kept, h


# ---------------------------------------------------------------------------
# KK reconstruction (rx:170-244)
# ---------------------------------------------------------------------------

def hilbert_mult(nfft: int, delay: int) -> np.ndarray:
    k = np.arange(nfft // 2 + 1)
    mult = np.full(nfft // 2 + 1, -1j, dtype=np.complex128)
    mult[0] = 0.0
    mult[-1] = 0.0
    return mult * np.exp(-2j * np.pi * k * delay / nfft)


def kk_reconstruct(x: np.ndarray, nfft: int = 1024, state: dict | None = None,
                   clamp_rel: float = 1e-12):
    """Returns (field complex128[len(x)], new_state, diag) like rx:184-244."""
    hop = nfft // 2
    half = hop // 2
    x = np.asarray(x, dtype=np.float64)
    if len(x) == 0 or len(x) % hop:
        raise ValueError("chunk length must be a positive multiple of hop")
    if state is None:
        state = {"u_tail": np.zeros(hop), "a_hist": np.zeros(half),
                 "dead_hist": np.zeros(half, dtype=bool)}
    hops = x.reshape(-1, hop)
    mean = hops.mean(axis=1)
    dead = mean <= 0.0
    thr = np.where(dead, 1.0, clamp_rel * np.abs(mean))
    clamped = int(np.sum((hops < thr[:, None]) & ~dead[:, None]))
    safe = np.maximum(hops, thr[:, None])
    safe[dead] = 1.0
    flat = safe.reshape(-1)
    amp = np.sqrt(flat)
    u = 0.5 * np.log(flat)
    dmask = np.repeat(dead, hop)
    blocks = sliding_window_view(np.concatenate([state["u_tail"], u]), nfft)[::hop]
    phi = np.fft.irfft(np.fft.rfft(blocks, axis=1) * hilbert_mult(nfft, half),
                       n=nfft, axis=1)[:, hop:].reshape(-1)
    a_d = np.concatenate([state["a_hist"], amp])[:len(x)]
    d_d = np.concatenate([state["dead_hist"], dmask])[:len(x)]
    out = a_d * np.exp(1j * phi)
    out[d_d] = 0.0
    new = {"u_tail": u[-hop:].copy(), "a_hist": amp[-half:].copy(),
           "dead_hist": dmask[-half:].copy()}
    return out, new, {"clamped": clamped, "zero_blocks": np.nonzero(dead)[0].tolist()}


def freq_shift(x: np.ndarray, delta_f: float, fs: float, start: int) -> np.ndarray:
    """sc:286-299 (including the delta_f == 0 and start == 0 shortcut)."""
    if delta_f == 0.0 and start == 0:
        return x.copy()
    n = np.arange(start, start + len(x), dtype=np.float64)
    return x * np.exp(2j * np.pi * delta_f * n / fs)


# ---------------------------------------------------------------------------
# symbol sync (rx:574-601), DDLMS (rx:510-545), demap (rx:548-567)
# ---------------------------------------------------------------------------

class OracleSyncError(RuntimeError):
    pass


def symbol_sync(y2: np.ndarray, ref: np.ndarray, min_ratio: float = 4.0):
    from scipy.signal import fftconvolve

    ref = np.asarray(ref, dtype=np.complex128)
    best = None
    for parity in (0, 1):
        z = y2[parity::2]
        if len(z) < len(ref):
            continue
        mag = np.abs(fftconvolve(z, np.conj(ref[::-1]), mode="valid"))
        k = int(np.argmax(mag))
        side = np.delete(mag, np.arange(max(0, k - 2), min(len(mag), k + 3)))
        rms = np.sqrt(np.mean(side ** 2)) if len(side) else 1e-30
        ratio = mag[k] / rms
        if best is None or ratio > best[2]:
            best = (parity, k, ratio)
    if best is None:
        raise OracleSyncError("stream shorter than the reference sequence")
    parity, k, ratio = best
    if ratio < min_ratio:
        raise OracleSyncError(f"no correlation peak (peak-to-rms {ratio:.2f})")
    return 2 * k + parity, float(ratio)


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "_build", "liboracle_ddlms.so")
        if not os.path.exists(path):
            subprocess.run(["make", "-s", "-C", HERE], check=True)
        lib = ctypes.CDLL(path)
        P = ctypes.c_void_p
        lib.oracle_ddlms_core.argtypes = [
            P, ctypes.c_int64, P, P, ctypes.c_int, P, ctypes.c_int, P, ctypes.c_int64,
            ctypes.c_double, ctypes.c_int, ctypes.c_double, ctypes.c_double,
            ctypes.c_int64, P, P, P, ctypes.c_int64]
        lib.oracle_ddlms_core.restype = ctypes.c_int
        _LIB = lib
    return _LIB


@dataclass
class EqState:
    w: np.ndarray
    g: np.ndarray
    resid: np.ndarray = field(default_factory=lambda: np.zeros(0, np.complex128))
    frozen: bool = False
    div_count: int = 0
    symbols_done: int = 0

    @classmethod
    def initial(cls, n_taps=4, spike=1):
        w = np.zeros(n_taps, np.complex128)
        w[spike] = 1.0
        return cls(w=w, g=np.zeros(n_taps, np.complex128))


def ddlms_wl(x, state: EqState, training=None, order=4, n_taps=4, mu=1e-3,
             widely_linear=True, guard_factor=10.0, guard_run=100):
    spec = constellation(order)
    xc = np.ascontiguousarray(np.concatenate([state.resid, np.asarray(x, np.complex128)]))
    n_out = max(0, (len(xc) - n_taps) // 2 + 1)
    soft = np.empty(n_out, np.complex128)
    dec = np.empty(n_out, np.complex128)
    train = (np.zeros(0, np.complex128) if training is None
             else np.ascontiguousarray(np.asarray(training, np.complex128)[:n_out]))
    if n_out:
        st = np.array([int(state.frozen), int(state.div_count)], dtype=np.int64)
        w = np.ascontiguousarray(state.w)
        g = np.ascontiguousarray(state.g)
        pts = np.ascontiguousarray(spec.points)
        _lib().oracle_ddlms_core(
            xc.ctypes.data, len(xc), w.ctypes.data, g.ctypes.data, n_taps,
            pts.ctypes.data, len(pts), train.ctypes.data, len(train), float(mu),
            int(bool(widely_linear)), spec.max_radius, float(guard_factor), int(guard_run),
            st.ctypes.data, soft.ctypes.data, dec.ctypes.data, n_out)
        state.w, state.g = w, g
        state.frozen, state.div_count = bool(st[0]), int(st[1])
    state.resid = xc[2 * n_out:].copy()
    state.symbols_done += n_out
    return dec, soft, state


def demap(symbols, order):
    spec = constellation(order)
    symbols = np.asarray(symbols, np.complex128)
    k = spec.bits_per_symbol
    shifts = np.arange(k - 1, -1, -1)
    bits = np.empty(len(symbols) * k, np.uint8)
    nfb = 0
    for a in range(0, len(symbols), 1 << 16):
        b = min(a + (1 << 16), len(symbols))
        d = np.abs(symbols[a:b, None] - spec.points[None, :])
        idx = np.argmin(d, axis=1)
        nfb += int(np.sum(d[np.arange(b - a), idx] > 1e-9))
        bits[a * k:b * k] = ((spec.labels[idx][:, None] >> shifts[None, :]) & 1).reshape(-1)
    return bits, nfb


# ---------------------------------------------------------------------------
# streaming pipeline (rx:608-815)
# ---------------------------------------------------------------------------

@dataclass
class OracleConfig:
    taps: np.ndarray                       # static taps @ adc_rate/2 (FirFilter)
    adc_rate_hz: float = 4e9
    tone_freq_hz: float = 0.516e9
    kk_fft: int = 1024
    static_fft: int = 32768
    carrier_removal: bool = True
    carrier_segment_len: int = 1 << 16
    mirror: bool = True
    aa_edge: float = 0.01
    n_taps: int = 4
    mu: float = 1e-3
    startup_symbols: int = 10_000
    widely_linear: bool = True
    divergence_factor: float = 10.0
    divergence_run: int = 100
    order: int = 4
    sync_symbols: int = 4096
    sync_wait_samples: int = 1 << 16


class OraclePipeline:
    """Chunk-streaming restatement of RxPipeline (rx:608-815)."""

    def __init__(self, cfg: OracleConfig, reference_symbols=None, record=False):
        self.cfg = cfg
        self.ref = None if reference_symbols is None else np.asarray(reference_symbols, np.complex128)
        self.aa_delay = cfg.static_fft // 4
        self.kept, self.resp = static_response(cfg.taps, cfg.adc_rate_hz / 2.0, cfg.static_fft,
                                               cfg.adc_rate_hz, cfg.aa_edge, self.aa_delay)
        self.raw = np.zeros(0)
        self.kk_state = None
        self.cfifo = np.zeros(0, np.complex128)
        self.ds_index = 0
        self.sfifo = np.zeros(0, np.complex128)
        self.stail = None
        self.eq = EqState.initial(cfg.n_taps)
        self.sync_buf = np.zeros(0, np.complex128)
        self.train_left = 0
        self.train_pos = 0
        self.synced = False
        self.eq_scale = None
        self.sync_offset = None
        self.sync_ratio = None
        self.decs, self.softs = [], []
        self.record = record
        self.rec = {"kk": [], "static": [], "ddlms_in": []}

    def _static(self, x, flush):
        cfg = self.cfg
        hop = cfg.static_fft // 2
        self.sfifo = np.concatenate([self.sfifo, x])
        if flush and len(self.sfifo) % hop:
            self.sfifo = np.concatenate([self.sfifo, np.zeros(hop - len(self.sfifo) % hop, np.complex128)])
        n_full = (len(self.sfifo) // hop) * hop
        if n_full == 0:
            return np.zeros(0, np.complex128)
        chunk, self.sfifo = self.sfifo[:n_full], self.sfifo[n_full:]
        if self.stail is None:
            self.stail = np.zeros(hop, np.complex128)
        n, m = cfg.static_fft, cfg.static_fft // 2
        blocks = sliding_window_view(np.concatenate([self.stail, chunk]), n)[::hop]
        y = np.fft.ifft(np.fft.fft(blocks, axis=1)[:, self.kept] * self.resp, axis=1) * (m / n)
        self.stail = chunk[-hop:].copy()
        return y[:, m // 2:].reshape(-1)

    def _ddlms(self, y2, flush):
        cfg = self.cfg
        if not self.synced:
            self.sync_buf = np.concatenate([self.sync_buf, y2])
            need = cfg.sync_wait_samples + 2 * cfg.sync_symbols
            if len(self.sync_buf) < need and not flush:
                return
            head = self.sync_buf[:need]
            skip = min(len(head) // 2, 1 << 13)
            rms = np.sqrt(np.mean(np.abs(head[skip:]) ** 2))
            self.eq_scale = 1.0 / rms if rms > 0 else 1.0
            drop = 0
            if self.ref is not None:
                off, ratio = symbol_sync(head, self.ref[:cfg.sync_symbols])
                self.sync_offset, self.sync_ratio = off, ratio
                drop = max(0, off - 1)
                self.train_left = min(cfg.startup_symbols, len(self.ref))
                self.train_pos = 0
            y2 = self.sync_buf[drop:]
            self.sync_buf = np.zeros(0, np.complex128)
            self.synced = True
        if len(y2) == 0:
            return
        y2 = y2 * self.eq_scale
        if self.record:
            self.rec["ddlms_in"].append(y2.copy())
        train = None
        if self.train_left > 0:
            train = self.ref[self.train_pos:self.train_pos + self.train_left]
        dec, soft, self.eq = ddlms_wl(
            y2, self.eq, train, order=cfg.order, n_taps=cfg.n_taps, mu=cfg.mu,
            widely_linear=cfg.widely_linear, guard_factor=cfg.divergence_factor,
            guard_run=cfg.divergence_run)
        if self.train_left > 0:
            used = min(len(dec), self.train_left)
            self.train_left -= used
            self.train_pos += used
        self.decs.append(dec)
        self.softs.append(soft)

    def feed(self, x, flush=False):
        cfg = self.cfg
        hop = cfg.kk_fft // 2
        self.raw = np.concatenate([self.raw, np.asarray(x, np.float64)])
        if flush and len(self.raw) % hop:
            self.raw = np.concatenate([self.raw, np.zeros(hop - len(self.raw) % hop)])
        n_full = (len(self.raw) // hop) * hop
        if n_full == 0 and not flush:
            return
        chunk, self.raw = self.raw[:n_full], self.raw[n_full:]
        if len(chunk):
            field_, self.kk_state, _ = kk_reconstruct(chunk, cfg.kk_fft, self.kk_state)
        else:
            field_ = np.zeros(0, np.complex128)
        if self.record:
            self.rec["kk"].append(field_.copy())
        # carrier removal on the global segment grid (rx:671-688)
        if cfg.carrier_removal:
            self.cfifo = np.concatenate([self.cfifo, field_])
            seg = cfg.carrier_segment_len
            take = len(self.cfifo) if flush else (len(self.cfifo) // seg) * seg
            cl = self.cfifo[:take].copy()
            self.cfifo = self.cfifo[take:]
            for a in range(0, take, seg):
                cl[a:a + seg] -= np.mean(cl[a:a + seg])
        else:
            cl = field_
        # downshift with the global index + mirror (rx:690-696, rx:247-257)
        sh = freq_shift(cl, -cfg.tone_freq_hz, cfg.adc_rate_hz, self.ds_index) \
            if not (cfg.tone_freq_hz == 0 and self.ds_index == 0) else cl.copy()
        self.ds_index += len(cl)
        if cfg.mirror:
            sh = np.conj(sh)
        y2 = self._static(sh, flush)
        if self.record:
            self.rec["static"].append(y2.copy())
        self._ddlms(y2, flush)

    def drain(self):
        d = np.concatenate(self.decs) if self.decs else np.zeros(0, np.complex128)
        s = np.concatenate(self.softs) if self.softs else np.zeros(0, np.complex128)
        self.decs, self.softs = [], []
        return d, s

    def finish(self):
        self.feed(np.zeros(0), flush=True)
        return self.drain()


def receive(adc: np.ndarray, cfg: OracleConfig, ref_symbols, buffer_len: int, record=False):
    """hr:94-101 receive_stream + finish."""
    pipe = OraclePipeline(cfg, ref_symbols, record=record)
    for a in range(0, len(adc), buffer_len):
        pipe.feed(adc[a:a + buffer_len])
    dec, soft = pipe.finish()
    return pipe, dec, soft


# ---------------------------------------------------------------------------
# BER (hr:104-137 measure_point; me:69-130)
# ---------------------------------------------------------------------------

def q_from_ber(ber: float) -> float:
    from scipy.special import erfcinv
    if ber == 0:
        return float("inf")
    return float(20.0 * np.log10(np.sqrt(2.0) * erfcinv(2.0 * ber)))


def count_errors_aligned(dec_idx: np.ndarray, sym_idx: np.ndarray, order: int,
                         start: int, stop: int) -> tuple[int, int]:
    """Bit errors of decisions [start, stop) against transmitted symbols at
    the same indices (the alignment frame_sync finds at me:97-112 when the
    pipeline synchronised)."""
    spec = constellation(order)
    k = spec.bits_per_symbol
    a = spec.labels[dec_idx[start:stop]]
    b = spec.labels[sym_idx[start:stop]]
    x = np.bitwise_xor(a, b)
    errs = int(sum(int(np.sum((x >> s) & 1)) for s in range(k)))
    return errs, (stop - start) * k


def to_index(values: np.ndarray, order: int) -> np.ndarray:
    pts = constellation(order).points
    return np.argmin(np.abs(np.asarray(values)[:, None] - pts[None, :]), axis=1).astype(np.uint8)


# ---------------------------------------------------------------------------
# fiber span, split-step Fourier (channel.py ssfm_span :124-158, cd
# coefficient :80-85) -- the step before the receive path;
# pinned to kkmodem by tests/golden/channel_ssfm.npz (tools/gen_golden_channel.py)
# ---------------------------------------------------------------------------
def cd_phase_coefficient(dispersion_ps_nm_km: float, length_km: float, lambda_nm: float) -> float:
    d_si = dispersion_ps_nm_km * 1e-6
    lam = lambda_nm * 1e-9
    return np.pi * d_si * lam ** 2 * (length_km * 1e3) / 299792458.0


def ssfm_span(samples: np.ndarray, fs: float, length_km: float, loss_db_per_km: float, dispersion_ps_nm_km: float,
              gamma_per_w_km: float, step_km: float | None = None, lambda_nm: float = 1550.116) -> np.ndarray:
    if step_km is None:
        step_km = 1.0
    if step_km <= 0:
        raise ValueError("step_km must be positive")
    step_km = min(step_km, length_km) if length_km > 0 else step_km
    n_steps = max(1, int(round(length_km / step_km)))
    dz = length_km / n_steps
    alpha = loss_db_per_km * np.log(10.0) / 10.0
    a_half = cd_phase_coefficient(dispersion_ps_nm_km, dz / 2.0, lambda_nm)
    f = np.fft.fftfreq(len(samples), 1.0 / fs)
    lin_half = np.exp(-1j * a_half * f * f)
    l_eff = (1.0 - np.exp(-alpha * dz)) / alpha if alpha > 0 else dz
    loss_amp = np.exp(-alpha * dz / 2.0)
    x = np.asarray(samples, dtype=np.complex128).copy()
    for _ in range(n_steps):
        x = np.fft.ifft(np.fft.fft(x) * lin_half)
        x = x * np.exp(1j * gamma_per_w_km * (np.abs(x) ** 2 * 1e-3) * l_eff)
        x = np.fft.ifft(np.fft.fft(x) * lin_half)
        x *= loss_amp
    return x
