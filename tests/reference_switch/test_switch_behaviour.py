"""Run INSIDE the reference-suite subprocess (tests/test_reference_suite.py),
with the kkmodem backend switch installed (-p paper_2108_07001_b200.kkmodem_backend):
checks that the reference's own callers handle the B200 receiver's errors
and objects exactly as they handle kkmodem's.  Not collected by the main
suite (tests/conftest.py collect_ignore)."""

import numpy as np
import pytest

import kkmodem.rxdsp as krx
import kkmodem.sigcore as ksc
from kkmodem.harness.config import preset
from kkmodem.harness.runner import run_single

import paper_2108_07001_b200.rxdsp as gpu
from paper_2108_07001_b200 import kkmodem_backend


def test_switch_installed():
    assert kkmodem_backend.installed()
    assert krx.RxPipeline is gpu.RxPipeline
    import kkmodem.harness.runner as krun
    assert krun.RxPipeline is gpu.RxPipeline and krun.demap is gpu.demap


def test_errors_are_kkmodems():
    assert issubclass(gpu.SyncError, krx.SyncError)
    assert issubclass(gpu.ParameterError, ksc.ParameterError)
    with pytest.raises(ksc.ParameterError):
        krx.kk_reconstruct(ksc.RealSignal(np.ones(1000), 4e9), ksc.BlockPlan(1024, buffer_len=1 << 13))
    rng = np.random.default_rng(14)
    noise = rng.standard_normal(20000) + 1j * rng.standard_normal(20000)
    ref = np.exp(0.5j * np.pi * rng.integers(0, 4, 2000))     # unrelated to the noise
    with pytest.raises(krx.SyncError):
        krx.symbol_sync(noise, ref)


def test_pipeline_accepts_kkmodem_realsignal():
    cfg = krx.RxPipelineConfig()
    pipe = krx.RxPipeline(cfg)
    pipe.feed(ksc.RealSignal(np.full(1 << 14, 4.0), 4e9))
    assert pipe.samples_in == 1 << 14


def test_forced_sync_failure_marks_point_failed():
    """runner.py:182-184: a SyncError raised by the (GPU) pipeline marks the
    point failed and the run continues.  Forced with an OSNR override far
    below the payload, so the training correlation has no peak."""
    cfg = preset("ci")
    cfg.tx.n_symbols = 1 << 15
    cfg.tx.cspr_db = 12.0
    cfg.link.n_spans = 1
    cfg.link.span_length_km = 0.0
    cfg.link.ase_enabled = False
    cfg.link.phase_noise_linewidth_hz = 0.0
    cfg.link.monitor_every_n_spans = 1
    cfg.rx.sync_wait_samples = 1 << 14
    cfg.rx.startup_symbols = 4000
    cfg.rx.osnr_override_db = -30.0
    report = run_single(cfg)
    (point,) = report["points"]
    assert point["status"] == "failed", point
    assert "peak" in point["reason"] or "correlation" in point["reason"], point["reason"]


def test_nonlinear_link_runs_gpu_spans():
    """channel.py:208-209: propagate_link calls ssfm_span by name, so with the
    switch the nonlinear spans are the GPU split-step (kk_ssfm_span); its
    output equals the reference's own span to float64 rounding."""
    import kkmodem.channel as kch
    from paper_2108_07001_b200 import channel as gch

    assert kch.ssfm_span is gch.ssfm_span
    orig = kkmodem_backend._saved[("ch", "ssfm_span")]
    rng = np.random.default_rng(8)
    x = ksc.ComplexSignal(np.sqrt(5.0) * (rng.standard_normal(6000) + 1j * rng.standard_normal(6000)), 16e9)
    span = kch.FiberSpan(length_km=100.0)
    got = kch.ssfm_span(x, span, 10.0)
    want = orig(x, span, 10.0)
    assert type(got) is type(want)
    err = np.linalg.norm(got.samples - want.samples) / np.linalg.norm(want.samples)
    assert err < 1e-10, err
