"""The oracle (oracle/kkoracle.py) pinned against the REAL reference's outputs
stored in tests/golden/ (tools/gen_golden.py ran kkmodem's RxPipeline /
measure_point on these exact ADC streams).  CPU only."""

import json
import os

import numpy as np
import pytest

from oracle import kkoracle as ko

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
NAMES = sorted(f[:-5] for f in os.listdir(GOLDEN) if f.endswith(".json"))


def load(name):
    with open(os.path.join(GOLDEN, name + ".json")) as f:
        meta = json.load(f)
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    return meta, {k: z[k] for k in z.files}


def oracle_run(meta, arr, reps=1):
    x = arr["adc_h"].astype(np.float64) * (meta["lsb"] / 2.0)
    syms = ko.constellation(meta["order"]).points[arr["sym_idx"]]
    if reps > 1:
        x, syms = np.tile(x, reps), np.tile(syms, reps)
    cfg = ko.OracleConfig(taps=arr["taps"], order=meta["order"], mu=meta["mu"],
                          startup_symbols=meta["startup_symbols"])
    return ko.receive(x, cfg, syms, meta["buffer_len"], record=True)


def test_goldens_present():
    assert len(NAMES) >= 12


@pytest.mark.parametrize("name", NAMES)
def test_oracle_reproduces_reference(name):
    meta, arr = load(name)
    pipe, dec, soft = oracle_run(meta, arr)
    assert pipe.sync_offset == meta["sync_offset"]
    assert pipe.sync_ratio == pytest.approx(meta["sync_ratio"], rel=1e-12)
    assert pipe.eq_scale == pytest.approx(meta["eq_scale"], rel=1e-13)   # static output within 1e-9: ulp-level
    assert len(dec) == meta["n_dec"]
    idx = ko.to_index(dec, meta["order"])
    assert np.array_equal(idx, arr["dec_idx"])                 # bit-exact decisions
    sh = arr["soft_head"]
    assert np.max(np.abs(soft[: len(sh)].astype(np.complex64) - sh)) <= 1e-6
    # BER over measure_point's region (runner.py:109-118) with the aligned count
    head = meta["startup_symbols"] + meta["head_guard_symbols"]
    stop = len(dec) - meta["tail_guard_symbols"]
    e, n = ko.count_errors_aligned(idx, arr["sym_idx"], meta["order"], head, stop)
    assert e == meta["point"]["n_errors"]
    assert n == meta["point"]["n_bits"]
    if "kk_prefix" in arr:
        kk = np.concatenate(pipe.rec["kk"])[: len(arr["kk_prefix"])]
        assert np.max(np.abs(kk.astype(np.complex64) - arr["kk_prefix"])) == 0.0
        st = np.concatenate(pipe.rec["static"])[: len(arr["static_prefix"])]
        assert np.max(np.abs(st.astype(np.complex64) - arr["static_prefix"])) < 1e-9


@pytest.mark.parametrize("name", ["c5_qpsk_10000km_tile", "c3_64qam_1600km_tile"])
def test_oracle_tiled_stream(name):
    meta, arr = load(name)
    pipe, dec, _ = oracle_run(meta, arr, reps=meta["tile_reps"])
    assert pipe.sync_offset == meta["sync_offset4"]
    assert np.array_equal(ko.to_index(dec, meta["order"]), arr["dec4_idx"])


def test_oracle_chunking_invariant():
    meta, arr = load("c1_qpsk_b2b")
    x = arr["adc_h"].astype(np.float64) * (meta["lsb"] / 2.0)
    syms = ko.constellation(4).points[arr["sym_idx"]]
    cfg = ko.OracleConfig(taps=arr["taps"])
    _, d1, s1 = ko.receive(x, cfg, syms, len(x))
    p = ko.OraclePipeline(cfg, syms)
    rng = np.random.default_rng(0)
    prev = 0
    for c in list(np.sort(rng.integers(1, len(x), 7))) + [len(x)]:
        p.feed(x[prev:c])
        prev = c
    d2, s2 = p.finish()
    assert np.array_equal(d1, d2) and np.array_equal(s1, s2)


def test_oracle_kk_constant_and_zero_block():
    out, _, dg = ko.kk_reconstruct(np.full(1 << 14, 4.0))
    assert np.allclose(out[2048:-2048], 2.0, rtol=1e-12)
    x = np.ones(1 << 13)
    x[512:1024] = 0.0
    out, _, dg = ko.kk_reconstruct(x)
    assert dg["zero_blocks"] == [1]
    assert np.all(out[768:1280] == 0)


def _ssfm_cases():
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "channel_ssfm.npz"))
    out = []
    i = 0
    while f"x{i}" in z:
        n, fs, L, loss, D, g, step, p = z[f"p{i}"]
        out.append((z[f"x{i}"], z[f"y{i}"], dict(fs=fs, length_km=L, loss_db_per_km=loss, dispersion_ps_nm_km=D,
                                                 gamma_per_w_km=g, step_km=None if np.isnan(step) else step)))
        i += 1
    return out


def test_oracle_ssfm_span_reproduces_reference():
    """The split-step span restatement (channel.py:124-158) equals kkmodem's
    own ssfm_span on the golden inputs (same numpy calls and order)."""
    cases = _ssfm_cases()
    assert len(cases) == 4
    for x, y, kw in cases:
        got = ko.ssfm_span(x, **kw)
        assert np.array_equal(got, y)
