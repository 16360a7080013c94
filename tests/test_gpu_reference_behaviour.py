"""The reference's own behavioural criteria for the receive stages
(kkmodem tests/test_rxdsp.py), restated against the B200 implementation:
the same inputs and pass/fail bars, expressed with this package's API (the
reference package itself does not travel to the GPU box).  Where the B200
path computes in fp32 the tolerance is stated next to the reference's."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2108_07001_b200 import rxdsp  # noqa: E402
from paper_2108_07001_b200.constellation import make_constellation  # noqa: E402
from paper_2108_07001_b200.sigcore import BlockPlan, ComplexSignal, FirFilter, ParameterError, RealSignal, design_rrc  # noqa: E402,E501


def _ideal_2sps_qpsk(n_symbols, seed, sps=2):
    """Clean 2-sps QPSK at the symbol peaks, RRC cascade collapsed
    (test_rxdsp.py:257-270): random bits -> Gray QPSK points, raised cosine."""
    rng = np.random.default_rng(seed)
    spec = make_constellation(4)
    syms = spec.points[rng.integers(0, 4, n_symbols)]
    rrc = design_rrc(0.01, sps, 256).taps.real
    rc = np.convolve(rrc, rrc)
    x = np.zeros(n_symbols * sps, dtype=complex)
    x[::sps] = syms
    y = np.convolve(x, rc)
    d = len(rc) // 2
    return syms, y[d:d + n_symbols * sps]


def _mp_waveform(n_symbols=1 << 14, cspr_db=12.0, seed=0, order=4, tone_hz=0.516e9):
    """Minimum-phase test field at 4 GS/s (test_rxdsp.py:36-47 restated):
    random symbols, RRC (rolloff 0.01, span 256) shaping at 4 sps scaled by
    sqrt(sps) and trimmed causally (txdsp.py:220-234), plus a tone at
    +tone_hz with amplitude sqrt(P * 10^(CSPR/10)) (txdsp.py:242-249)."""
    from scipy.signal import fftconvolve

    rng = np.random.default_rng(seed)
    syms = make_constellation(order).points[rng.integers(0, order, n_symbols)]
    sps = 4
    rrc = design_rrc(0.01, sps, 256).taps.real
    x = np.zeros(n_symbols * sps, dtype=complex)
    x[::sps] = syms
    wave = fftconvolve(x, rrc)[:len(x)] * np.sqrt(sps)
    amp = np.sqrt(np.mean(np.abs(wave) ** 2) * 10.0 ** (cspr_db / 10.0))
    n = np.arange(len(wave))
    return wave, wave + amp * np.exp(2j * np.pi * tone_hz * n / 4e9)


def _true_mp_field(payload, tone_hz, cspr_db, fs=4e9):
    """test_rxdsp.py:50-57: tone amplitude at DC plus the mirrored payload."""
    n = np.arange(len(payload))
    amp = np.sqrt(np.mean(np.abs(payload) ** 2) * 10 ** (cspr_db / 10))
    return amp + np.conj(payload) * np.exp(2j * np.pi * tone_hz * n / fs)


def _kk_error(cspr_db, n_symbols, seed):
    wave, field = _mp_waveform(n_symbols, cspr_db=cspr_db, seed=seed)
    plan = BlockPlan(1024, buffer_len=len(field))
    rec, _, _ = rxdsp.kk_reconstruct(RealSignal(np.abs(field) ** 2, 4e9), plan)
    target = _true_mp_field(wave, 0.516e9, cspr_db)
    d = plan.hop // 2                                     # emitted with hop/2 delay
    sl = slice(4096, len(target) - 4096 - d)
    err = np.asarray(rec.samples)[d:][sl] - target[sl]
    return np.mean(np.abs(err) ** 2), np.mean(np.abs(target[sl]) ** 2)


def test_kk_mp_reconstruction_error():
    """test_rxdsp.py:91-103 (construction oracle): KK of a known
    minimum-phase field at CSPR 12 dB is within -30 dB of the analytic target."""
    e, p = _kk_error(12.0, 1 << 14, 1)
    assert 10 * np.log10(e / p) < -30.0


def test_kk_error_monotone_in_cspr():
    """test_rxdsp.py:105-115: the reconstruction error falls as CSPR rises."""
    errs = [_kk_error(c, 1 << 13, 2)[0] for c in (4.0, 6.0, 8.0, 10.0, 12.0)]
    assert all(a >= b for a, b in zip(errs, errs[1:])), errs


def test_downshift_zero_is_identity_and_inverse_pair():
    """test_rxdsp.py:132-141: a zero shift is the identity; +f then -f
    restores the signal (float64 phase on the device, rtol 1e-12)."""
    sig = ComplexSignal(np.exp(1j * np.arange(256)), 4e9)
    assert np.array_equal(rxdsp.downshift_dc(sig, 0.0).samples, sig.samples)
    rng = np.random.default_rng(2)
    sig = ComplexSignal(rng.standard_normal(1024) + 1j * rng.standard_normal(1024), 4e9)
    out = rxdsp.downshift_dc(rxdsp.downshift_dc(sig, 0.516e9), -0.516e9)
    assert np.allclose(out.samples, sig.samples, rtol=1e-12)


def test_payload_centered_after_kk():
    """test_rxdsp.py:143-156 (PSD-centroid oracle): KK reconstruction of the
    minimum-phase test field, mean removed, downshifted by the tone: the
    payload PSD centroid within +-0.6 GHz lies within 5 MHz of DC."""
    _, field = _mp_waveform(seed=3)
    plan = BlockPlan(1024, buffer_len=len(field))
    rec, _, _ = rxdsp.kk_reconstruct(RealSignal(np.abs(field) ** 2, 4e9), plan)
    s = np.asarray(rec.samples)
    shifted = rxdsp.downshift_dc(ComplexSignal(s - np.mean(s), 4e9), 0.516e9)
    trimmed = np.asarray(shifted.samples)[4096:-4096]
    psd = np.abs(np.fft.fft(trimmed)) ** 2
    f = np.fft.fftfreq(len(psd), 1 / 4e9)
    band = np.abs(f) < 0.6e9
    centroid = np.sum(f[band] * psd[band]) / np.sum(psd[band])
    assert abs(centroid) < 5e6, centroid


def test_static_allpass_is_decimation():
    """test_rxdsp.py:202-219: with a delta tap the static stage is a pure
    2:1 decimation of a signal band-limited inside the kept half band,
    delayed by aa_delay/2 output samples.  Oracle: x[::2] (exact for that
    band).  Reference bar 1e-6 (float64); fp32 FFT chain here: 1e-5."""
    rng = np.random.default_rng(4)
    n = 1 << 18
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    spec = np.fft.fft(x)
    f = np.fft.fftfreq(n, 1 / 4e9)
    spec[np.abs(f) > 0.9e9] = 0
    x = np.fft.ifft(spec)
    plan = BlockPlan(32768, buffer_len=1 << 18)
    out, _ = rxdsp.static_equalize_and_resample(ComplexSignal(x, 4e9), FirFilter(np.array([1.0 + 0j]), 2e9), plan)
    delay = plan.fft_size // 8
    a = np.asarray(out.samples)[delay + 4096:-4096]
    b = x[::2][4096:len(a) + 4096]
    err = np.linalg.norm(a - b) / np.linalg.norm(b)
    assert err < 1e-5, err


def test_static_output_rate_and_tap_rate_check():
    """test_rxdsp.py:244-255: output at half the rate, half the length; taps
    at the wrong rate raise ParameterError."""
    plan = BlockPlan(32768, buffer_len=1 << 18)
    sig = ComplexSignal(np.zeros(1 << 16, dtype=complex) + 1.0, 4e9)
    out, _ = rxdsp.static_equalize_and_resample(sig, FirFilter(np.array([1.0 + 0j]), 2e9), plan)
    assert out.sample_rate_hz == pytest.approx(2e9)
    assert len(out.samples) == (1 << 16) // 2
    with pytest.raises(ParameterError):
        rxdsp.static_equalize_and_resample(ComplexSignal(np.ones(1 << 16, dtype=complex), 4e9),
                                           FirFilter(np.ones(3), 4e9), plan)


def test_ddlms_qpsk_convergence():
    """test_rxdsp.py:273-285: clean QPSK, 5000 training symbols, mu 3e-3:
    every tail decision correct, tail MSE below -25 dB, no divergence."""
    syms, y2 = _ideal_2sps_qpsk(50000, seed=6)
    cfg = rxdsp.DdlmsConfig(mu=3e-3, startup_symbols=5000)
    dec, soft, state = rxdsp.ddlms_wl(y2, cfg, rxdsp.EqualizerState.initial(), training=syms,
                                      constellation=make_constellation(4))
    sl = slice(30000, len(syms) - 10)
    assert np.allclose(dec[sl], syms[sl])
    assert 10 * np.log10(np.mean(np.abs(soft[sl] - syms[sl]) ** 2)) < -25.0
    assert not state.diverged


def test_ddlms_widely_linear_corrects_conjugate_crosstalk():
    """test_rxdsp.py:287-305 (controlled-impairment A/B): x = 0.9 s + 0.1
    conj(s); the widely-linear equaliser makes no symbol errors and its error
    power is at least 10x below the strictly linear one's."""
    syms, y2 = _ideal_2sps_qpsk(60000, seed=7)
    x = 0.9 * y2 + 0.1 * np.conj(y2)
    spec = make_constellation(4)

    def run(widely):
        cfg = rxdsp.DdlmsConfig(mu=3e-3, startup_symbols=8000, widely_linear=widely)
        dec, soft, _ = rxdsp.ddlms_wl(x, cfg, rxdsp.EqualizerState.initial(), training=syms, constellation=spec)
        sl = slice(30000, len(syms) - 10)
        return np.mean(np.abs(soft[sl] - syms[sl]) ** 2), int(np.sum(dec[sl] != syms[sl]))

    err_wl, sym_err_wl = run(True)
    err_lin, _ = run(False)
    assert sym_err_wl == 0
    assert err_lin >= 10 * err_wl


# --- the reference runner's criteria (kkmodem tests/test_harness.py:99-163) ----

def _small_b2b(n_symbols=1 << 15):
    """small_b2b_config (test_harness.py:24-33) on the dict layout: the
    back-to-back QPSK golden config, shorter, faster sync/training."""
    import copy

    from paper_2108_07001_b200.captures import load_capture

    c = copy.deepcopy(load_capture("c1_qpsk_b2b").meta["config"])
    c["tx"]["n_symbols"] = n_symbols
    c["rx"]["sync_wait_samples"] = 1 << 14
    c["rx"]["startup_symbols"] = 4000
    return c


def test_run_single_noiseless_loopback_ber_zero():
    """test_harness.py:100-106: a noiseless back-to-back run decodes without
    a single bit error (BER 0, Q infinite)."""
    from paper_2108_07001_b200.harness import run_single

    (point,) = run_single(_small_b2b())["points"]
    assert point["status"] == "ok" and point["ber"] == 0.0 and point["q_db"] == np.inf


def test_run_single_monitors_and_deterministic_reports(tmp_path):
    """test_harness.py:108-130: a 10-span link monitored every 2 spans
    reports at 200..1000 km; two runs of the same config write
    byte-identical reports."""
    from paper_2108_07001_b200.harness import run_single

    c = _small_b2b()
    c["link"].update(n_spans=10, span_length_km=100.0, monitor_every_n_spans=2, ase_enabled=True)
    rep = run_single(c, output_dir=str(tmp_path / "a"))
    assert [p["distance_km"] for p in rep["points"]] == [200.0, 400.0, 600.0, 800.0, 1000.0]
    run_single(c, output_dir=str(tmp_path / "b"))
    assert (tmp_path / "a" / "report.json").read_bytes() == (tmp_path / "b" / "report.json").read_bytes()


def test_run_sweep_rows_and_csv(tmp_path):
    """test_harness.py:133-157: values x monitored distances rows, the CSV
    with a header, the optimum file; a one-value sweep succeeds."""
    from paper_2108_07001_b200.harness import run_sweep

    c = _small_b2b()
    c["link"].update(n_spans=2, span_length_km=100.0, monitor_every_n_spans=1, ase_enabled=True)
    c["sweep"] = {"axis": "cspr_db", "values": [8.0, 10.0, 12.0]}
    res = run_sweep(c, output_dir=str(tmp_path))
    assert len(res["rows"]) == 3 * 2
    assert len((tmp_path / "sweep.csv").read_text().strip().splitlines()) == 1 + 6
    assert (tmp_path / "sweep_optimum.csv").exists()
    c1 = _small_b2b()
    c1["sweep"] = {"axis": "cspr_db", "values": [12.0]}
    res1 = run_sweep(c1)
    assert len(res1["rows"]) == 1 and res1["rows"][0]["status"] == "ok"
