"""Generate the golden fixtures under tests/golden/ from the REAL reference.

Test infrastructure only: this script imports the reference package
(`kkmodem`, installed into baseline/_ref or copied from /root/reference) in
THIS container, replays the reference's own `run_single` data path
(`harness/runner.py:148-169`: build_transmit_side -> wiener_phase_noise ->
propagate_link -> photodetect -> adc_quantize), and records

* the ADC stream as exact int16 odd half-LSB codes h (value = h * lsb/2;
  `frontend.py:108-117` mid-rise levels (code+0.5)*lsb),
* the transmitted symbols (as constellation indices) and bits,
* the reference receiver's outputs (`RxPipeline` fed per buffer exactly as
  `receive_stream` `runner.py:94-101`, then `finish`): decisions, soft
  symbols (a slice), sync offset/ratio, eq scale, the `measure_point`
  BER/EVM report (`runner.py:104-137`),
* per-stage intermediates (KK field, carrier-removed field, downshifted,
  2-sps static output) for a prefix of the stream.

The fixtures are small compressed .npz files plus one JSON index.  Nothing on
the GPU box reads /root/reference: it only reads these committed fixtures.

Usage:  python tools/gen_golden.py [--only NAME ...]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
OUT = os.path.join(REPO, "tests", "golden")


def _import_reference():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
    cand = [os.path.join(REPO, "baseline", "_ref")]
    for c in cand:
        if os.path.isdir(os.path.join(c, "kkmodem")):
            sys.path.insert(0, c)
            break
    else:
        import shutil
        dst = "/tmp/kkmodem_ref_copy"
        if not os.path.isdir(dst):
            shutil.copytree("/root/reference/pkg/src", dst)
        sys.path.insert(0, dst)
    import kkmodem  # noqa: F401
    return kkmodem


kkmodem = _import_reference()
from kkmodem.channel import propagate_link, wiener_phase_noise  # noqa: E402
from kkmodem.frontend import adc_quantize, photodetect, super_gaussian_lowpass  # noqa: E402
from kkmodem.harness.config import preset  # noqa: E402
from kkmodem.harness.runner import (  # noqa: E402
    _derive_seeds, build_transmit_side, make_pipeline_config, measure_point,
)
from kkmodem.rxdsp import RxPipeline  # noqa: E402
from kkmodem.sigcore import RealSignal, resample_rational  # noqa: E402
from kkmodem.txdsp import make_constellation  # noqa: E402


# ---------------------------------------------------------------------------
# configurations (BASELINE.json configs)
# ---------------------------------------------------------------------------

def cfg_b2b(n_symbols=1 << 16, cspr_db=12.0):
    """Config 1: pkg/tests/test_harness.py:24-33 small_b2b_config."""
    cfg = preset("ci")
    cfg.tx.n_symbols = n_symbols
    cfg.tx.cspr_db = cspr_db
    cfg.link.n_spans = 1
    cfg.link.span_length_km = 0.0
    cfg.link.ase_enabled = False
    cfg.link.phase_noise_linewidth_hz = 0.0
    cfg.link.monitor_every_n_spans = 1
    return cfg


def cfg_link(order, n_spans, rel_db, cspr_db=10.0, n_symbols=1 << 16):
    """Configs 2-5: preset('ci') + n_spans x 100 km, one monitor at the end."""
    cfg = preset("ci")
    cfg.tx.n_symbols = n_symbols
    cfg.tx.constellation_order = order
    cfg.tx.cspr_db = cspr_db
    cfg.link.n_spans = n_spans
    cfg.link.monitor_every_n_spans = n_spans
    cfg.link.rel_launch_db = rel_db
    return cfg


CONFIGS = {
    "c1_qpsk_b2b": (cfg_b2b, {}),
    "c2_16qam_5600km_rel-20": (cfg_link, dict(order=16, n_spans=56, rel_db=-20.0)),
    "c2_16qam_5600km_rel-24": (cfg_link, dict(order=16, n_spans=56, rel_db=-24.0)),
    "c3_64qam_1600km_rel-20": (cfg_link, dict(order=64, n_spans=16, rel_db=-20.0)),
    "c3_64qam_1600km_rel-24": (cfg_link, dict(order=64, n_spans=16, rel_db=-24.0)),
}
for _c in (4.0, 6.0, 8.0, 10.0, 12.0, 14.0):
    CONFIGS[f"c4_qpsk_10000km_cspr{int(_c)}"] = (
        cfg_link, dict(order=4, n_spans=100, rel_db=-26.0, cspr_db=_c))
# Config 5 tile: 262,000 symbols = 1,048,000 ADC samples = 1048 x 1000, so the
# 0.516 GHz tone (129/1000 cycles per ADC sample) is phase-continuous across
# tile seams.
CONFIGS["c5_qpsk_10000km_tile"] = (
    cfg_link, dict(order=4, n_spans=100, rel_db=-26.0, cspr_db=10.0, n_symbols=262_000))

# 64-QAM 1,600 km tile (BASELINE configs[2]) for the bench's second format:
# same k*1000-sample tiling rule
CONFIGS["c3_64qam_1600km_tile"] = (
    cfg_link, dict(order=64, n_spans=16, rel_db=-20.0, cspr_db=10.0, n_symbols=262_000))

PREFIX = 1 << 15          # ADC samples of per-stage intermediates kept
SOFT_KEEP = 1 << 12       # soft symbols kept (head and tail) for soft-value parity
# configs that also carry per-stage intermediates (size budget)
STAGE_GOLDEN = {"c1_qpsk_b2b", "c3_64qam_1600km_rel-20", "c4_qpsk_10000km_cspr10"}


def capture(cfg):
    """Replay run_single's data path (runner.py:148-166) to the ADC stream."""
    seeds = _derive_seeds(cfg.seed)
    link = cfg.link.build()
    bits, syms, field = build_transmit_side(cfg)
    if link.phase_noise_linewidth_hz > 0:
        field = wiener_phase_noise(field, link.phase_noise_linewidth_hz,
                                   seed=seeds["phase_noise"])
    _, monitors = propagate_link(field, link, seed=seeds["link"])
    dist = sorted(monitors)[-1]
    sig = monitors[dist]
    fe = cfg.frontend
    current = photodetect(sig, fe)
    adc, clip = adc_quantize(current, fe, seed=seeds["electrical"])
    # recover the exact mid-rise codes: same arithmetic as frontend.py:95-117
    x = super_gaussian_lowpass(current.samples, current.sample_rate_hz,
                               fe.adc_analog_bandwidth_hz, fe.adc_aa_order)
    ratio = int(round(current.sample_rate_hz / fe.adc_rate_hz))
    s = resample_rational(RealSignal(x, current.sample_rate_hz), 1, ratio).samples
    rms = np.sqrt(np.mean(s ** 2))
    full_scale = 3.0 * rms
    n_levels = 1 << fe.adc_bits
    lsb = 2.0 * full_scale / n_levels
    codes = np.clip(np.floor(s / lsb), -n_levels // 2, n_levels // 2 - 1)
    h = (2 * codes + 1).astype(np.int16)
    assert np.array_equal(h.astype(np.float64) * (lsb / 2.0), adc.samples), "code recovery"
    return dict(bits=bits, syms=syms, adc=adc, h=h, lsb=lsb, link=link,
                dist=dist, clip=clip)


class RecordingPipeline(RxPipeline):
    """RxPipeline that records each stage's output (rxdsp.py:660-764)."""

    def __init__(self, *a, **k):
        super().__init__(*a, **k)
        self.rec = {"kk": [], "carrier": [], "downshift": [], "static": [], "ddlms_in": []}

    def _run_kk(self, x):
        out = super()._run_kk(x)
        self.rec["kk"].append(out.copy())
        return out

    def _run_carrier(self, x, flush):
        out = super()._run_carrier(x, flush)
        self.rec["carrier"].append(out.copy())
        return out

    def _run_downshift(self, x):
        out = super()._run_downshift(x)
        self.rec["downshift"].append(out.copy())
        return out

    def _run_static(self, x, flush):
        out = super()._run_static(x, flush)
        self.rec["static"].append(out.copy())
        return out


def receive(adc_samples, pipe_cfg, syms, record=False):
    cls = RecordingPipeline if record else RxPipeline
    pipe = cls(pipe_cfg, reference_symbols=syms)
    blen = pipe_cfg.kk_plan.buffer_len
    for start in range(0, len(adc_samples), blen):   # runner.py:99-100
        pipe.feed(adc_samples[start:start + blen])
    dec, soft = pipe.finish()
    return pipe, dec, soft


def to_index(values, spec):
    d = np.abs(values[:, None] - spec.points[None, :])
    idx = np.argmin(d, axis=1)
    assert np.max(d[np.arange(len(values)), idx]) < 1e-12
    return idx.astype(np.uint8)


def gen_one(name):
    fn, kw = CONFIGS[name]
    cfg = fn(**kw)
    t0 = time.time()
    cap = capture(cfg)
    t1 = time.time()
    pipe_cfg = make_pipeline_config(cfg, cap["link"])
    pipe, dec, soft = receive(cap["adc"].samples, pipe_cfg, cap["syms"], record=True)
    t2 = time.time()
    point = measure_point(dec, soft, cap["bits"], cap["syms"], cfg)
    spec = make_constellation(cfg.tx.constellation_order)
    cat = {k: np.concatenate(v) if v else np.zeros(0, complex) for k, v in pipe.rec.items()}
    arrays = dict(
        adc_h=cap["h"],
        sym_idx=to_index(cap["syms"], spec),
        bits_packed=np.packbits(cap["bits"]),
        taps=pipe_cfg.static_taps.taps,
        dec_idx=to_index(dec, spec),
        soft_head=soft[:SOFT_KEEP].astype(np.complex64),
        soft_tail=soft[-SOFT_KEEP:].astype(np.complex64),
    )
    if name in STAGE_GOLDEN:
        # the carrier/downshift stages are re-derived from kk_prefix in tests
        arrays["kk_prefix"] = cat["kk"][:PREFIX].astype(np.complex64)
        arrays["static_prefix"] = cat["static"][:PREFIX // 2].astype(np.complex64)
    meta = dict(
        name=name,
        n_symbols=cfg.tx.n_symbols,
        n_bits=int(len(cap["bits"])),
        order=cfg.tx.constellation_order,
        cspr_db=cfg.tx.cspr_db,
        n_spans=cfg.link.n_spans,
        distance_km=float(cap["dist"]),
        rel_launch_db=cfg.link.rel_launch_db,
        lsb=float(cap["lsb"]),
        adc_len=int(len(cap["h"])),
        clip_fraction=float(cap["clip"]),
        buffer_len=pipe_cfg.kk_plan.buffer_len,
        mu=pipe_cfg.ddlms.mu,
        startup_symbols=pipe_cfg.ddlms.startup_symbols,
        widely_linear=pipe_cfg.ddlms.widely_linear,
        sync_symbols=pipe_cfg.sync_symbols,
        sync_wait_samples=pipe_cfg.sync_wait_samples,
        tone_freq_hz=pipe_cfg.tone_freq_hz,
        n_dec=int(len(dec)),
        sync_offset=int(pipe.sync_offset),
        sync_ratio=float(pipe.sync_ratio),
        eq_scale=float(pipe._eq_scale),
        diverged=bool(pipe.diverged),
        stage_counts={k: int(len(v)) for k, v in cat.items()},
        diagnostics=pipe.diagnostics,
        point={k: v for k, v in point.items() if k != "windowed_q"},
        head_guard_symbols=cfg.metrics.head_guard_symbols,
        tail_guard_symbols=cfg.metrics.tail_guard_symbols,
        gen_seconds=round(t1 - t0, 2),
        rx_seconds=round(t2 - t1, 2),
        config=cfg.to_dict(),
    )
    if name.endswith("_tile"):
        # reference decisions on a 4-tile stream (the bench stream pattern,
        # runner.py:389-391 np.tile) -- checks seams end to end
        reps = 4
        stream = np.tile(cap["adc"].samples, reps)
        ref = np.tile(cap["syms"], reps)
        p4, d4, _ = receive(stream, pipe_cfg, ref)
        arrays["dec4_idx"] = to_index(d4, spec)
        meta["tile_reps"] = reps
        meta["n_dec4"] = int(len(d4))
        meta["sync_offset4"] = int(p4.sync_offset)
    path = os.path.join(OUT, f"{name}.npz")
    np.savez_compressed(path, **arrays)
    with open(os.path.join(OUT, f"{name}.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True, default=float)
    print(f"{name}: gen {t1 - t0:.1f}s rx {t2 - t1:.1f}s  dec={len(dec)} "
          f"ber={point['ber']:.3e} off={pipe.sync_offset} -> {os.path.getsize(path)/1e6:.2f} MB",
          flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*")
    args = ap.parse_args()
    os.makedirs(OUT, exist_ok=True)
    names = args.only or list(CONFIGS)
    for n in names:
        gen_one(n)


if __name__ == "__main__":
    main()
