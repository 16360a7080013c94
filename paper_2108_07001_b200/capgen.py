"""GPU capture generator -- the step before the receive path (SURVEY.md
§8(f)2): transmitter, linear fiber link, direct-detection front end and the
12-bit ADC, chunked so that arbitrarily long physical captures (2^30 ADC
samples of a 10,000 km link) are produced on the device instead of tiling a
short reference capture.

Reference stages it restates (kkmodem):
  bits      prbs_generate tx:180-205 (two-tap Fibonacci LFSR, taps tx:33)
  symbols   qam_map tx:208-217 (Gray labels of make_constellation tx:115-142)
  shaping   shape tx:220-234 (unit-energy RRC x sqrt(sps), causal, trimmed)
  carrier   add_carrier tx:237-244 (tone at +tone_freq, amplitude from CSPR)
  phase     wiener_phase_noise ch:207-217 (increment variance 2 pi lw / fs)
  link      propagate_link ch:189-204: per span CD + loss, EDFA restoring the
            launch power with ASE (ch:162-186); nonlinearity off (the
            shipped configs 1-5)
  frontend  photodetect fe:84-100 (flat-top OBPF, |E|^2, super-Gaussian PD
            low-pass), adc_quantize fe:103-118 (super-Gaussian AA low-pass,
            decimation, mid-rise 12-bit quantizer at 3x RMS full scale)

B200 design: one overlap-save pipeline at the simulation rate, its FFTs the
repo's float64 transforms (channel.fft / ifft -> kk_fft, batched rows):
  A  shaping FIR straight at the simulation rate (sps_sim = fs / baud), the
     carrier tone (exact rational phase) and the Wiener phase (carried);
  B  FFT(field) * CD(total length) + FFT(ASE) -> * OBPF -> IFFT, where the
     ASE of the N amplifiers is one white Gaussian stream with their summed
     density (CD and the EDFA gains are linear and all-pass, so the sum is
     white with the same total variance; equal in distribution);
  C  |y|^2, FFT * (PD x AA super-Gaussian low-passes) -> IFFT -> every
     (fs / adc_rate)-th sample (the AA response is ~2^-128 at the ADC
     Nyquist, so the decimation does not alias);
  D  mid-rise quantizer to the exact int16 wire format (odd half-LSB codes).
Differences from the reference (deliberate, documented): linear (overlap-
save) instead of whole-capture circular filtering, shaping directly at the
simulation rate instead of at the DAC rate + FFT resampling, and ASE drawn
with torch's Philox generator -- so captures agree statistically (EVM, BER,
sync offset), not sample for sample.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .constellation import make_constellation
from .sigcore import AdcCodes, ParameterError, cd_phase_coefficient, design_rrc

# two-tap Fibonacci LFSR taps per degree (the reference's table, tx:33)
PRBS_TAPS = {7: (6, 7), 15: (14, 15), 23: (18, 23), 31: (28, 31)}

_C = 299792458.0


def _fft(x, n=None):
    """FFT over the last axis (zero padded to n) on kk_fft."""
    import torch

    from .channel import fft
    if n is not None and x.shape[-1] < n:
        x = torch.cat([x, x.new_zeros(*x.shape[:-1], n - x.shape[-1])], -1)
    return fft(x.contiguous())


def _ifft(x):
    from .channel import ifft
    return ifft(x.contiguous())
_H = 6.62607015e-34


def prbs_bits(degree: int, seed: int, n: int) -> np.ndarray:
    """Maximal-length PRBS bits: b[k] = b[k - a] ^ b[k - b] after the seed
    state (bit i of the seed value as b[i]); one period is generated and
    repeated (uint8 0/1)."""
    if degree not in PRBS_TAPS:
        raise ParameterError(f"PRBS degree must be one of {sorted(PRBS_TAPS)}")
    if seed == 0:
        raise ParameterError("PRBS seed must be nonzero")
    a, b = PRBS_TAPS[degree]
    period = (1 << degree) - 1
    s = (abs(int(seed)) - 1) % period + 1
    m = min(n, period)
    buf = np.empty(m + degree, dtype=np.uint8)
    buf[:degree] = (s >> np.arange(degree)) & 1
    # b[k] = b[k-a] ^ b[k-b] implies b[k] = b[k - a 2^j] ^ b[k - b 2^j] for
    # k >= b 2^j (the connection polynomial squared j times over GF(2)):
    # grow the prefix in vectorised steps of a 2^j
    k, j = degree, 0
    while k < len(buf):
        while (b << (j + 1)) <= k:
            j += 1
        A, Bq = a << j, b << j
        step = min(A, len(buf) - k)
        buf[k:k + step] = buf[k - A:k - A + step] ^ buf[k - Bq:k - Bq + step]
        k += step
    one = buf[degree:degree + m]
    if n <= period:
        return one.copy()
    return np.resize(one, n)


def map_symbols(bits: np.ndarray, order: int) -> np.ndarray:
    """Bits (MSB first per symbol) -> constellation point indices (uint8)."""
    spec = make_constellation(order)
    k = spec.bits_per_symbol
    if len(bits) % k:
        raise ParameterError(f"bit count must be a multiple of {k}")
    w = (1 << np.arange(k - 1, -1, -1)).astype(np.int64)
    labels = np.asarray(bits, np.int64).reshape(-1, k) @ w
    return spec.label_to_index()[labels].astype(np.uint8)


@dataclass
class GenParams:
    baud_hz: float
    rolloff: float
    tone_freq_hz: float
    cspr_db: float
    order: int
    prbs_degree: int
    prbs_seed: int
    pulse_span_symbols: int
    sim_rate_hz: float
    launch_dbm: float
    n_spans: int
    span_km: float
    dispersion_ps_nm_km: float
    loss_db_per_km: float
    nf_db: float
    lambda_nm: float
    linewidth_hz: float
    ase_enabled: bool
    obpf_hz: float
    pd_hz: float
    pd_order: int
    adc_rate_hz: float
    adc_bits: int
    aa_hz: float
    aa_order: int
    # OSNR noise loading of the streaming back-to-back front end (runner.py
    # _StreamingFrontend, hr:257-264) instead of per-span ASE; None: off
    osnr_db: float | None = None
    obpf_enabled: bool = True

    @classmethod
    def from_config(cls, c: dict) -> "GenParams":
        """From an experiment config dict (harness.config.ExperimentConfig.to_dict
        layout, as stored in the golden captures' metadata)."""
        tx, ln, fe = c["tx"], c["link"], c["frontend"]
        if ln.get("nonlinearity_enabled"):
            raise ParameterError("the GPU generator models the linear link only")
        return cls(baud_hz=tx["baud_hz"], rolloff=tx["rolloff"], tone_freq_hz=tx["tone_freq_hz"],
                   cspr_db=tx["cspr_db"], order=tx["constellation_order"], prbs_degree=tx["prbs_degree"],
                   prbs_seed=tx["prbs_seed"], pulse_span_symbols=tx["pulse_span_symbols"],
                   sim_rate_hz=c["sim_rate_hz"], launch_dbm=ln["total_launch_dbm"] + ln["rel_launch_db"],
                   n_spans=ln["n_spans"], span_km=ln["span_length_km"],
                   dispersion_ps_nm_km=ln["dispersion_ps_nm_km"], loss_db_per_km=ln["loss_db_per_km"],
                   nf_db=ln["edfa_noise_figure_db"], lambda_nm=ln["center_wavelength_nm"],
                   linewidth_hz=ln["phase_noise_linewidth_hz"], ase_enabled=ln["ase_enabled"],
                   obpf_hz=fe["obpf_bandwidth_hz"], pd_hz=fe["pd_bandwidth_hz"], pd_order=fe["pd_filter_order"],
                   adc_rate_hz=fe["adc_rate_hz"], adc_bits=fe["adc_bits"], aa_hz=fe["adc_analog_bandwidth_hz"],
                   aa_order=fe["adc_aa_order"])

    def ase_sigma2_mw(self) -> float:
        """Total ASE power (mW over the simulation bandwidth) of the N EDFAs
        (ch:162-186: gain restores the launch power after each span)."""
        if not self.ase_enabled:
            return 0.0
        g = 10.0 ** (self.loss_db_per_km * self.span_km / 10.0)
        if g <= 1.0:
            return 0.0
        nf = 10.0 ** (self.nf_db / 10.0)
        nsp = (g * nf - 1.0) / (2.0 * (g - 1.0))
        nu = _C / (self.lambda_nm * 1e-9)
        return self.n_spans * (g - 1.0) * nsp * _H * nu * self.sim_rate_hz * 1e3


class CaptureGenerator:
    """Chunked GPU generator of an int16 ADC capture (see module doc)."""

    def __init__(self, params: GenParams, seed: int = 0, device=None, block: int = 1 << 16):
        import torch

        self.p = p = params
        self.dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        fs = p.sim_rate_hz
        sps = fs / p.baud_hz
        if abs(sps - round(sps)) > 1e-9:
            raise ParameterError("simulation rate must be a multiple of the baud rate")
        self.sps = int(round(sps))
        dec = fs / p.adc_rate_hz
        if abs(dec - round(dec)) > 1e-9:
            raise ParameterError("simulation rate must be a multiple of the ADC rate")
        self.dec = int(round(dec))
        tone = p.tone_freq_hz / fs
        from fractions import Fraction
        fr = Fraction(tone).limit_denominator(1 << 20)
        if abs(float(fr) - tone) > 1e-15:
            raise ParameterError("tone frequency must be a rational fraction of the simulation rate")
        self.tone_p, self.tone_q = fr.numerator, fr.denominator
        self.gen = torch.Generator(device=self.dev)
        self.gen.manual_seed(int(seed))
        # shaping FIR at the simulation rate (unit energy x sqrt(sps): unit mean power)
        rrc = design_rrc(p.rolloff, self.sps, p.pulse_span_symbols).taps.real * np.sqrt(self.sps)
        self.rrc = torch.from_numpy(rrc).to(self.dev, torch.float32)
        self.n_fir = len(rrc)
        # optical block filter: CD over the whole link x flat-top OBPF
        self.N = int(block)
        self.ov = 4096                          # overlap (CD spread ~25 ns = 400 samples at 16 GS/s)
        f = np.fft.fftfreq(self.N, 1.0 / fs)
        a = cd_phase_coefficient(p.dispersion_ps_nm_km, p.n_spans * p.span_km, p.lambda_nm)
        cd = np.exp(-1j * a * f * f)
        half = p.obpf_hz / 2.0
        fp = half * 0.95
        af = np.abs(f)
        ob = np.where(af <= fp, 1.0, np.where(af < half, 0.5 * (1 + np.cos(np.pi * (af - fp) / (half - fp))), 0.0))
        if not p.obpf_enabled:
            ob = np.ones_like(af)
        # the zero-phase / symmetric responses are delayed by half the overlap
        # so they are causal inside the overlap-save window
        delay = np.exp(-2j * np.pi * f * (self.ov // 2) / fs)
        self.H_cd = torch.from_numpy(cd).to(self.dev, torch.complex64)
        self.H_ob = torch.from_numpy(ob * delay).to(self.dev, torch.complex64)
        # electrical block filter: PD x AA super-Gaussians (the AA response is
        # ~2^-128 at the ADC Nyquist: plain decimation does not alias)
        el = np.exp(-0.5 * np.log(2.0) * (f / p.pd_hz) ** (2 * p.pd_order))
        el = el * np.exp(-0.5 * np.log(2.0) * (f / p.aa_hz) ** (2 * p.aa_order))
        self.H_el = torch.from_numpy(el * delay).to(self.dev, torch.complex64)
        k = make_constellation(p.order).bits_per_symbol
        self.period_bits = prbs_bits(p.prbs_degree, p.prbs_seed, (1 << p.prbs_degree) - 1)
        self.bits_per_symbol = k
        # streaming state
        self.sym_pos = 0
        self.sim_pos = 0
        self.theta = 0.0
        self.fir_tail = torch.zeros(self.n_fir - 1, dtype=torch.complex64, device=self.dev)
        self.opt_tail = torch.zeros(2, self.ov, dtype=torch.complex64, device=self.dev)
        self.el_tail = torch.zeros(self.ov, dtype=torch.complex64, device=self.dev)
        self.scale_sig = None
        self.full_scale = None

    # -- stage A: shaping + carrier + laser phase noise -----------------------
    def _transmit(self, sym_c):
        import torch

        p, sps = self.p, self.sps
        n = sym_c.shape[0] * sps
        x = torch.zeros(n, dtype=torch.complex64, device=self.dev)
        x[::sps] = sym_c
        xx = torch.cat([self.fir_tail, x])
        L = 1 << int(np.ceil(np.log2(len(xx) + self.n_fir)))
        y = _ifft(_fft(xx, L) * _fft(self.rrc.to(torch.complex64), L)).to(torch.complex64)
        y = y[self.n_fir - 1:self.n_fir - 1 + n]              # causal linear convolution, chunk part
        self.fir_tail = xx[-(self.n_fir - 1):]
        if self.scale_sig is None:                             # amplitudes frozen on the first chunk
            ps = float(torch.mean(y.abs() ** 2))
            self.amp_tone = np.sqrt(ps * 10.0 ** (p.cspr_db / 10.0))
            launch_mw = 10.0 ** (p.launch_dbm / 10.0)
            tot = ps + self.amp_tone ** 2
            self.scale_sig = np.sqrt(launch_mw / tot)
            sig2 = p.ase_sigma2_mw()
            # EDFAs restore the total power: signal share shrinks by the noise share
            self.scale_sig *= np.sqrt(max(launch_mw - sig2, 0.0) / launch_mw)
            self.noise_std = np.sqrt(sig2 / 2.0)
            if p.osnr_db is not None:
                # white field noise at the OSNR (12.5 GHz reference bandwidth)
                # relative to the total (signal + carrier) power, hr:257-264
                density = ps * (1.0 + 10.0 ** (p.cspr_db / 10.0)) / (10.0 ** (p.osnr_db / 10.0) * 12.5e9)
                self.noise_std = np.sqrt(density * p.sim_rate_hz / 2.0) * self.scale_sig
        k = torch.arange(self.sim_pos, self.sim_pos + n, device=self.dev, dtype=torch.int64)
        ph = 2.0 * np.pi * ((k * self.tone_p) % self.tone_q).to(torch.float64) / self.tone_q
        field = y + (self.amp_tone * torch.polar(torch.ones_like(ph), ph)).to(torch.complex64)
        if p.linewidth_hz > 0:
            sig = np.sqrt(2.0 * np.pi * p.linewidth_hz / p.sim_rate_hz)
            inc = torch.randn(n, generator=self.gen, device=self.dev, dtype=torch.float64) * sig
            th = torch.cumsum(inc, 0) + self.theta
            self.theta = float(th[-1])
            field = field * torch.polar(torch.ones_like(th), th).to(torch.complex64)
        self.sim_pos += n
        return field * self.scale_sig

    # -- overlap-save block filtering with a carried tail -----------------------
    def generate(self, n_symbols: int, chunk_symbols: int = 1 << 18):
        """A whole capture: (int16 wire codes on the device, half_lsb, point
        indices (host), bits (host)); the quantizer scale is frozen on the
        first chunk, so the codes are one consistent stream."""
        import torch

        codes, idx, bits = [], [], []
        half = None
        done = 0
        while done < n_symbols:
            m = min(chunk_symbols, n_symbols - done)
            a, i, b = self.next_chunk(m)
            codes.append(a.codes)
            idx.append(i)
            bits.append(b)
            half = a.half_lsb
            done += m
        return torch.cat(codes), half, np.concatenate(idx), np.concatenate(bits)

    def _ols(self, xx, n):
        """Overlap-save blocks of the stream xx (..., ov + n): (..., nblk, N)
        views (zero-padded at the end), all transformed in one batched FFT."""
        import torch

        hop = self.N - self.ov
        nblk = -(-n // hop)
        need = self.ov + nblk * hop + (self.N - hop - self.ov)
        if xx.shape[-1] < need:
            xx = torch.nn.functional.pad(xx, (0, need - xx.shape[-1]))
        return _fft(xx.unfold(-1, self.N, hop)).to(torch.complex64)

    def _ols_out(self, Y, n):
        import torch

        y = _ifft(Y).to(torch.complex64)[..., self.ov:]
        return y.reshape(*y.shape[:-2], -1)[..., :n]

    def next_chunk(self, n_symbols: int):
        """(AdcCodes of 4 * n_symbols ADC samples (int16 on the device),
        transmitted point indices (uint8, host), bits (uint8, host))."""
        import torch

        p = self.p
        k = self.bits_per_symbol
        per = self.period_bits
        b0 = (self.sym_pos * k) % len(per)
        bits = np.take(per, np.arange(b0, b0 + n_symbols * k) % len(per))
        idx = map_symbols(bits, p.order)
        pts = torch.from_numpy(make_constellation(p.order).points).to(self.dev, torch.complex64)
        field = self._transmit(pts[torch.from_numpy(idx.astype(np.int64)).to(self.dev)])
        self.sym_pos += n_symbols
        n = field.shape[0]
        if self.noise_std > 0:
            noise = torch.complex(torch.randn(n, generator=self.gen, device=self.dev),
                                  torch.randn(n, generator=self.gen, device=self.dev)) * float(self.noise_std)
        else:
            noise = torch.zeros_like(field)
        # B: CD on the field, ASE added, OBPF on both (one batched FFT)
        xx = torch.cat([self.opt_tail, torch.stack([field, noise])], 1)
        F = self._ols(xx, n)
        opt = self._ols_out((F[0] * self.H_cd + F[1]) * self.H_ob, n)
        self.opt_tail = xx[:, -self.ov:]
        # C: photodiode |E|^2, electrical response, decimation
        cur = (opt.abs() ** 2).to(torch.complex64)
        xe = torch.cat([self.el_tail, cur])
        el = self._ols_out(self._ols(xe, n) * self.H_el, n).real
        self.el_tail = xe[-self.ov:]
        adc = el[::self.dec].to(torch.float64)
        # D: 12-bit mid-rise quantizer, full scale 3 x RMS (frozen on the first chunk)
        if self.full_scale is None:
            self.full_scale = 3.0 * float(torch.sqrt(torch.mean(adc[adc.shape[0] // 2:] ** 2)))
        nl = 1 << p.adc_bits
        lsb = 2.0 * self.full_scale / nl
        codes = torch.clamp(torch.floor(adc / lsb), -(nl // 2), nl // 2 - 1)
        wire = (2 * codes + 1).to(torch.int16)                    # odd half-LSB codes
        return AdcCodes(wire, lsb / 2.0, p.adc_rate_hz), idx, bits
