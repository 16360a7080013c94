"""Host-side logic of the drop-in package (no GPU): constellation tables and
slicer descriptors, plans/config validation, receive-tap design (checked
against the taps the reference designed for each golden capture), metrics
helpers and super-frame planning."""

import numpy as np
import pytest

from oracle import kkoracle as ko
from paper_2108_07001_b200 import rxdsp
from paper_2108_07001_b200.captures import list_captures, load_capture
from paper_2108_07001_b200.constellation import make_constellation, slicer_tables
from paper_2108_07001_b200.metrics import frame_sync, q_from_ber, windowed_q
from paper_2108_07001_b200.sigcore import BlockPlan, FirFilter, ParameterError, RealSignal
from paper_2108_07001_b200.superframe import HALO_SAMPLES, plan_superframe


@pytest.mark.parametrize("order", [4, 8, 16, 32, 64])
def test_constellations_match_oracle(order):
    a, b = make_constellation(order), ko.constellation(order)
    assert np.array_equal(a.points, b.points) and np.array_equal(a.labels, b.labels)


@pytest.mark.parametrize("order", [4, 16, 64])
def test_square_slicer_grid(order):
    tb = slicer_tables(order)
    assert tb.grid_m == int(np.sqrt(order))
    pts = make_constellation(order).points
    rng = np.random.default_rng(order)
    y = (rng.standard_normal(5000) + 1j * rng.standard_normal(5000)) * 1.2
    # the separable rule used on the GPU == the reference's argmin
    v_r = np.clip(np.rint(y.real * tb.norm / 2 + (tb.grid_m - 1) / 2), 0, tb.grid_m - 1).astype(int)
    v_i = np.clip(np.rint(y.imag * tb.norm / 2 + (tb.grid_m - 1) / 2), 0, tb.grid_m - 1).astype(int)
    sep = tb.grid[v_r * tb.grid_m + v_i]
    brute = np.argmin(np.abs(y[:, None] - pts[None, :]), axis=1)
    assert np.array_equal(sep, brute)


def test_non_square_use_brute_force():
    for order in (8, 32):
        assert slicer_tables(order).grid_m == 0


def test_plans_and_config_validation():
    assert BlockPlan(1024, buffer_len=1 << 22).blocks_per_buffer == 8192
    with pytest.raises(ParameterError):
        BlockPlan(1000)
    with pytest.raises(ParameterError):
        rxdsp.RxPipelineConfig(baud_hz=2e9)
    with pytest.raises(ParameterError):
        rxdsp.RxPipelineConfig(static_taps=FirFilter(np.ones(4), 2e9))


def test_stream_buffers():
    plan = BlockPlan(1024, buffer_len=4096)
    bufs = list(rxdsp.stream_buffers(RealSignal(np.ones(5000), 4e9), plan))
    assert len(bufs) == 2
    assert bufs[1]["n_padding"] == 4096 - (5000 - 4096)
    assert np.array_equal(bufs[0]["tail"], np.zeros(512))
    with pytest.raises(ParameterError):
        list(rxdsp.stream_buffers(RealSignal(np.ones(100), 4e9), plan))


class _NS:
    def __init__(self, **kw):
        self.__dict__.update(kw)


def _link_tx_fe(meta):
    c = meta["config"]
    L = c["link"]
    link = _NS(total_dispersion_ps_nm=L["n_spans"] * L["span_length_km"] * L["dispersion_ps_nm_km"],
               center_wavelength_nm=L["center_wavelength_nm"])
    tx = _NS(**{k: c["tx"][k] for k in ("baud_hz", "rolloff", "pulse_span_symbols", "tone_freq_hz")})
    fe = _NS(**{k: c["frontend"][k] for k in ("pd_bandwidth_hz", "pd_filter_order", "adc_analog_bandwidth_hz",
                                               "adc_aa_order")})
    return link, tx, fe


@pytest.mark.parametrize("name", ["c1_qpsk_b2b", "c4_qpsk_10000km_cspr10", "c3_64qam_1600km_rel-20"])
def test_receive_tap_design_matches_reference(name):
    cap = load_capture(name)
    link, tx, fe = _link_tx_fe(cap.meta)
    fir = rxdsp.design_receive_taps(link, tx, frontend=fe, n_taps=203, rate_hz=2e9)
    assert np.max(np.abs(fir.taps - cap.taps)) < 1e-9 * np.max(np.abs(cap.taps))


def test_compute_static_taps_zero_link_is_delta():
    fir = rxdsp.compute_static_taps(_NS(total_dispersion_ps_nm=0.0, center_wavelength_nm=1550.0))
    c = len(fir.taps) // 2
    assert abs(fir.taps[c] - 1) < 1e-6 and np.max(np.abs(np.delete(fir.taps, c))) < 1e-6
    with pytest.raises(ParameterError):
        rxdsp.compute_static_taps(_NS(total_dispersion_ps_nm=0.0, center_wavelength_nm=1550.0), n_taps=202)


def test_static_response_matches_oracle():
    cap = load_capture("c4_qpsk_10000km_cspr10")
    kept, h = rxdsp._static_response(FirFilter(cap.taps, 2e9), BlockPlan(32768), 4e9, 0.01, 8192)
    k2, h2 = ko.static_response(cap.taps, 2e9, 32768, 4e9, 0.01, 8192)
    assert np.array_equal(kept, k2) and np.max(np.abs(h - h2)) < 1e-12


def test_metrics_helpers():
    assert q_from_ber(0) == np.inf
    assert q_from_ber(1e-3) == pytest.approx(ko.q_from_ber(1e-3))
    rng = np.random.default_rng(1)
    tx = rng.integers(0, 2, 1 << 15).astype(np.uint8)
    rx = tx[1000:20000].copy()
    off, a, b = frame_sync(rx, tx)
    assert off == 1000 and np.array_equal(a, b)
    q = windowed_q(np.zeros(10000, np.uint8), 1e6, 0.001)
    assert len(q) == 10 and all(v == q_from_ber(1e-3) for _, v in q)


def test_superframe_planning():
    n = 1 << 30
    jobs = [plan_superframe(r, 4, n) for r in range(4)]
    assert jobs[0].load_start == 0 and jobs[-1].load_end == 4 * n
    for j in jobs[1:]:
        assert j.core_start - j.load_start == HALO_SAMPLES
        assert j.load_start % 65536 == 0
    assert all(a.core_end == b.core_start for a, b in zip(jobs, jobs[1:]))


def test_captures_index():
    names = list_captures()
    assert "c5_qpsk_10000km_tile" in names
    cap = load_capture("c1_qpsk_b2b")
    assert cap.adc_h.dtype == np.int16 and np.all(cap.adc_h % 2 != 0)
    cfg = cap.pipeline_config()
    assert cfg.static_taps is not None and cfg.constellation_order == 4


def test_bench_throughput_needs_enough_samples():
    """runner.py:379-380 (test_harness.py:191-194): fewer than 4 buffers of
    samples raise ValueError before any work."""
    from paper_2108_07001_b200.harness import bench_throughput

    cfg = load_capture("c1_qpsk_b2b").meta["config"]
    with pytest.raises(ValueError):
        bench_throughput(cfg, n_samples=1 << 10)


def test_run_sweep_drives_the_reference_sweep(tmp_path, monkeypatch):
    """harness.run_sweep is the reference's own sweep driver (sweep.py:41-83:
    axis application, rows, argmax summary, CSVs) with run_single swapped for
    the GPU one -- here a stand-in returning a fixed report per point."""
    from paper_2108_07001_b200 import harness

    seen = []

    def fake_run_single(c):
        seen.append(c["tx"]["cspr_db"])
        q = 10.0 - abs(c["tx"]["cspr_db"] - 10.0)
        return {"points": [{"distance_km": 1e4, "status": "ok", "ber": 1e-3, "q_db": q, "evm_pct": 5.0,
                            "n_bits": 100, "n_errors": 1}]}

    monkeypatch.setattr(harness, "run_single", fake_run_single)
    c = load_capture("c4_qpsk_10000km_cspr10").meta["config"]
    c = dict(c, sweep={"axis": "cspr_db", "values": [6.0, 10.0, 14.0]})
    res = harness.run_sweep(c, output_dir=str(tmp_path))
    assert seen == [6.0, 10.0, 14.0]
    assert len(res["rows"]) == 3 and res["summary"][0]["best_value"] == 10.0
    assert (tmp_path / "sweep.csv").read_text().count("\n") == 4
    assert (tmp_path / "sweep_optimum.csv").exists()
    with pytest.raises(ValueError):                    # the reference's ParameterError
        harness.run_sweep(dict(c, sweep=None))


# --- the reference's host-side tap criteria (kkmodem test_rxdsp.py:158-385),
# restated against this package's float64 host setup code ---------------------

def _link_10000km():
    """LinkConfig() defaults: 100 x 100 km at 20 ps/nm/km, 1550.116 nm."""
    from types import SimpleNamespace

    return SimpleNamespace(total_dispersion_ps_nm=20.0 * 10000.0, center_wavelength_nm=1550.116)


def test_static_tap_coverage_and_even_taps():
    """test_rxdsp.py:168-172, :194-196: tap span covers the 10,000 km delay
    spread (the reference's units included); an even tap count is rejected."""
    assert rxdsp.static_tap_coverage(_link_10000km(), n_taps=203, rate_hz=2e9) > 10.0
    with pytest.raises(ParameterError):
        rxdsp.compute_static_taps(_link_10000km(), n_taps=202)


def test_static_taps_cascade_flat():
    """test_rxdsp.py:174-192 (cascade frequency-response oracle): taps x fiber
    CD is flat within 0.2 dB and 0.05 rad of linear phase over +-0.5 GHz."""
    from paper_2108_07001_b200.sigcore import cd_phase_coefficient, fir_frequency_response

    link = _link_10000km()
    fir = rxdsp.compute_static_taps(link, n_taps=203)
    f = np.linspace(-0.5e9, 0.5e9, 501)
    a = cd_phase_coefficient(link.total_dispersion_ps_nm, 1.0, link.center_wavelength_nm)
    cascade = fir_frequency_response(fir, f) * np.exp(-1j * a * f * f)
    mag_db = 20 * np.log10(np.abs(cascade))
    phase = np.unwrap(np.angle(cascade))
    resid = phase - np.polyval(np.polyfit(f, phase, 1), f)
    assert np.max(np.abs(mag_db - np.mean(mag_db))) < 0.2
    assert np.max(np.abs(resid)) < 0.05


def test_receive_taps_undo_dispersion():
    """test_rxdsp.py:359-375: TX pulse -> 10,000 km CD -> designed receive
    taps, sampled at the symbol period, has ISI below 3 %."""
    from types import SimpleNamespace

    from paper_2108_07001_b200.sigcore import cd_phase_coefficient, design_rrc

    link = _link_10000km()
    tx = SimpleNamespace(baud_hz=1e9, rolloff=0.01, pulse_span_symbols=256, tone_freq_hz=0.516e9)
    fir = rxdsp.design_receive_taps(link, tx)
    assert len(fir.taps) == 203
    pulse = design_rrc(0.01, 2, 256).taps.real
    x = np.concatenate([pulse, np.zeros(4096 - len(pulse))])
    f = np.fft.fftfreq(len(x), 1 / 2e9)
    a = cd_phase_coefficient(20.0, 10000.0, link.center_wavelength_nm)
    dispersed = np.fft.ifft(np.fft.fft(x) * np.exp(-1j * a * f * f))
    composite = np.convolve(dispersed, fir.taps)
    peak = int(np.argmax(np.abs(composite)))
    vals = np.abs(composite[peak % 2::2])
    ci = (peak - peak % 2) // 2
    assert np.sqrt(np.sum(np.delete(vals, ci) ** 2)) / vals[ci] < 0.03


def test_refine_static_taps_fits_capture():
    """test_rxdsp.py:377-384: the data-aided refit absorbs a mild unknown
    3-tap channel (relative MSE below 1e-2)."""
    from paper_2108_07001_b200.sigcore import design_rrc

    rng = np.random.default_rng(12)
    syms = make_constellation(4).points[rng.integers(0, 4, 6000)]
    rc = np.convolve(design_rrc(0.01, 2, 256).taps.real, design_rrc(0.01, 2, 256).taps.real)
    up = np.zeros(2 * len(syms), dtype=complex)
    up[::2] = syms
    y2 = np.convolve(up, rc)[len(rc) // 2:len(rc) // 2 + len(up)]
    x = np.convolve(y2, np.array([0.05 - 0.02j, 1.0, -0.08 + 0.03j]), mode="same")
    _, diag = rxdsp.refine_static_taps(x, syms, n_taps=31, rate_hz=2e9)
    assert diag["relative_mse"] < 1e-2


def test_pack12_round_trip_and_layout():
    """Packed 12-bit wire format (sigcore.AdcPacked12): exact round trip of
    odd half-LSB codes over the whole 12-bit range, the documented byte layout,
    and the contract errors."""
    from paper_2108_07001_b200.sigcore import AdcPacked12, pack12, unpack12

    c = np.arange(-2048, 2048)
    h = (2 * np.concatenate([c, c[::-1]]) + 1).astype(np.int16)
    p = pack12(h)
    assert len(p) == 3 * len(h) // 2
    assert np.array_equal(unpack12(p, len(h)), h)
    # layout: c0 = -2048 (0x800), c1 = 5 -> 0x00, 0x58, 0x00
    assert list(pack12(np.array([2 * -2048 + 1, 2 * 5 + 1], np.int16))) == [0x00, 0x58, 0x00]
    with pytest.raises(ParameterError):
        pack12(np.array([1, 2], np.int16))          # even code: not a mid-rise level
    with pytest.raises(ParameterError):
        AdcPacked12(p[:3], 1.0, 3)                  # odd sample count


def test_bench_refuses_more_gpus_than_visible():
    """bench.py --gpus N without torchrun self-launches N ranks, but refuses
    (exit 2, message) when fewer than N GPUs are visible; a WORLD_SIZE that
    differs from --gpus is refused too (no line may claim a GPU count it did
    not run on)."""
    import os
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    r = subprocess.run([sys.executable, os.path.join(repo, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 2, (r.returncode, r.stderr[-500:])
    assert "--gpus 2 requested" in r.stderr
    env["WORLD_SIZE"] = "1"
    r = subprocess.run([sys.executable, os.path.join(repo, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 2 and "WORLD_SIZE=1" in r.stderr
