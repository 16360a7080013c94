"""Callers of the receiver (kkmodem.harness.runner, cited `hr:line`) that
touch the hot path: pipeline construction, buffer-wise receive, BER/Q/EVM
measurement, and a device-resident streaming run.

`make_pipeline_config` accepts the reference's ExperimentConfig / LinkConfig
duck-typed (attributes tx, rx, link, frontend), so the reference harness,
sweeps and presets drive the B200 pipeline unchanged.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .constellation import make_constellation, slicer_tables
from .metrics import (SyncFailure, count_bit_errors, evm, frame_sync, q_from_ber, windowed_q,
                      windowed_q_from_counts)
from ._lib import SyncError
from .rxdsp import _upload, side_stream
from .rxdsp import (
    DdlmsConfig, GpuOptions, RxPipeline, RxPipelineConfig, compute_static_taps, demap, design_receive_taps,
)

from .sigcore import BlockPlan, ParameterError


def make_pipeline_config(cfg, link, gpu: GpuOptions | None = None) -> RxPipelineConfig:
    """hr:65-91."""
    rx, tx = cfg.rx, cfg.tx
    rate_out = cfg.frontend.adc_rate_hz / 2.0
    if rx.designed_taps:
        taps = design_receive_taps(link, tx, frontend=cfg.frontend if rx.compensate_frontend else None,
                                   n_taps=rx.static_n_taps, rate_hz=rate_out)
    else:
        taps = compute_static_taps(link, n_taps=rx.static_n_taps, rate_hz=rate_out)
    return RxPipelineConfig(
        adc_rate_hz=cfg.frontend.adc_rate_hz, baud_hz=tx.baud_hz, tone_freq_hz=tx.tone_freq_hz,
        kk_plan=BlockPlan(rx.kk_fft_size, buffer_len=rx.buffer_len),
        static_plan=BlockPlan(rx.static_fft_size, buffer_len=rx.buffer_len),
        static_taps=taps, carrier_removal=rx.carrier_removal, carrier_segment_len=rx.carrier_segment_len,
        ddlms=DdlmsConfig(mu=rx.mu, startup_symbols=rx.startup_symbols, widely_linear=rx.widely_linear),
        constellation_order=tx.constellation_order, sync_symbols=rx.sync_symbols,
        sync_wait_samples=rx.sync_wait_samples, gpu=gpu or GpuOptions())


def receive_stream(adc, pipe_cfg: RxPipelineConfig, reference_symbols) -> RxPipeline:
    """Feed a whole ADC stream buffer by buffer (hr:94-101)."""
    pipe = RxPipeline(pipe_cfg, reference_symbols=reference_symbols)
    x = adc.samples if hasattr(adc, "samples") else adc
    blen = pipe_cfg.kk_plan.buffer_len
    for start in range(0, len(x), blen):
        pipe.feed(x[start:start + blen])
    return pipe


def _namespace(d):
    """Attribute view of an ExperimentConfig.to_dict() layout."""
    from types import SimpleNamespace

    if isinstance(d, dict):
        return SimpleNamespace(**{k: _namespace(v) for k, v in d.items()})
    return d


def bench_throughput(cfg, n_samples: int, repeats: int = 3) -> dict:
    """Wall-clock throughput of the receiver chain over pre-generated input
    (runner.py:370-415, same arguments, errors and result keys).  `cfg` is an
    ExperimentConfig (anything with .to_dict()) or its dict layout.

    As in the reference, the input is a back-to-back capture of
    buffer_len/4 symbols tiled to n_samples (content does not change the
    arithmetic; the tiled decisions are meaningless).  Here the capture is
    generated on the GPU (capgen: the reference's TX/PD/ADC model) and stays
    resident in HBM as int16 wire codes; each repeat feeds it buffer by
    buffer through a fresh RxPipeline and finishes it (decisions returned to
    the host), timed with the device synchronised."""
    import copy
    import time

    import torch

    from . import capgen
    from .sigcore import AdcCodes

    c = copy.deepcopy(cfg.to_dict() if hasattr(cfg, "to_dict") else cfg)
    blen = int(c["rx"]["buffer_len"])
    if n_samples < 4 * blen:
        raise ValueError("need at least 4 buffers of samples")
    c["tx"]["n_symbols"] = blen // 4
    c["link"].update(n_spans=1, span_length_km=0.0, ase_enabled=False)
    gen = capgen.CaptureGenerator(capgen.GenParams.from_config(c), seed=int(c.get("seed", 0)))
    codes, half_lsb, idx, _ = gen.generate(blen // 4)
    reps = -(-n_samples // int(codes.shape[0]))
    stream = codes.repeat(reps)[:n_samples].contiguous()
    ref = make_constellation(c["tx"]["constellation_order"]).points[np.tile(idx, reps)[:n_samples // 4]]
    ns = _namespace(c)
    link = _namespace({"total_dispersion_ps_nm": 0.0, "center_wavelength_nm": c["link"]["center_wavelength_nm"]})
    pipe_cfg = make_pipeline_config(ns, link)
    results, last_pipe = [], None
    for _ in range(repeats):
        pipe = RxPipeline(pipe_cfg, reference_symbols=ref)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for start in range(0, n_samples, blen):
            pipe.feed(AdcCodes(stream[start:start + blen], half_lsb, pipe_cfg.adc_rate_hz))
        pipe.finish()
        torch.cuda.synchronize()
        elapsed = time.perf_counter() - t0
        results.append(n_samples / elapsed)
        last_pipe = pipe
    sps = float(np.median(results))
    stage = dict(last_pipe.stage_seconds)
    return {
        "samples_per_second": sps,
        "ratio_to_adc_rate": sps / float(c["frontend"]["adc_rate_hz"]),
        "repeats": results,
        "stage_seconds": stage,
        "stage_total_seconds": sum(stage.values()),
        "wall_seconds_last": n_samples / results[-1],
    }


REPORT_SCHEMA_VERSION = 1   # runner.py:38


def run_single(cfg, output_dir: str | None = None, save_captures: bool = False) -> dict:
    """tx -> link (with monitors) -> front end -> rx -> metrics (runner.py:
    140-196, same report schema: config echo and one point per monitored
    distance; a sync failure marks that point "failed").  The capture of
    each monitored distance is generated on the GPU (capgen: the reference's
    TX, linear link with per-span ASE and laser phase noise, PD and ADC;
    nonlinear links raise ParameterError) and received and measured on the
    device; noise realisations differ from the reference's, the statistics
    do not (test_capture_generator_statistics_vs_reference)."""
    import copy
    import json
    import os

    from . import capgen
    from .sigcore import AdcCodes, write_adc_raw

    c = copy.deepcopy(cfg.to_dict() if hasattr(cfg, "to_dict") else cfg)
    ln = c["link"]
    if ln.get("nonlinearity_enabled"):
        return _run_single_nonlinear(c, output_dir, save_captures)
    order = int(c["tx"]["constellation_order"])
    pts = make_constellation(order).points
    n_symbols = int(c["tx"]["n_symbols"])
    n_spans, every = int(ln["n_spans"]), max(1, int(ln["monitor_every_n_spans"]))
    monitors = [m for m in range(1, n_spans + 1) if m % every == 0 or m == n_spans]
    state = np.random.SeedSequence(int(c.get("seed", 0))).generate_state(4)          # hr:41-48
    link = _namespace({"total_dispersion_ps_nm": float(ln["dispersion_ps_nm_km"]) * n_spans
                       * float(ln["span_length_km"]), "center_wavelength_nm": ln["center_wavelength_nm"]})
    ns = _namespace(c)
    pipe_cfg = make_pipeline_config(ns, link)
    points = []
    for m in monitors:
        dist = m * float(ln["span_length_km"])
        point = {"distance_km": dist, "status": "ok"}
        cm = copy.deepcopy(c)
        cm["link"]["n_spans"] = m
        gp = capgen.GenParams.from_config(cm)
        gp.osnr_db = c["rx"].get("osnr_override_db")
        gen = capgen.CaptureGenerator(gp, seed=int(state[0]))
        codes, half, idx, bits = gen.generate(n_symbols)
        try:
            pipe = RxPipeline(pipe_cfg, reference_symbols=pts[idx])
            pipe.feed(AdcCodes(codes, half, pipe_cfg.adc_rate_hz))
            pipe.feed(np.zeros(0), flush=True)
            lab, soft, _ = pipe.drain_device()
            point.update(measure_point_device(lab, soft, bits, pts[idx], ns))
            full = (1 << int(c["frontend"]["adc_bits"])) - 1          # odd codes at the clip levels
            point["clip_fraction"] = float((codes.abs() >= full).float().mean())
            point["diverged"] = pipe.diverged
            if save_captures and output_dir:
                ddir = os.path.join(output_dir, f"dist_{int(dist):06d}km")
                os.makedirs(ddir, exist_ok=True)
                spec = make_constellation(order)
                k = spec.bits_per_symbol
                li = lab.cpu().numpy()
                li = np.where(li == 255, idx[:len(li)], li)
                pl = slicer_tables(order).point_label[:order]
                dbits = np.unpackbits(pl[li][:, None], axis=1)[:, -k:].reshape(-1)
                np.packbits(dbits).tofile(os.path.join(ddir, "decided_bits.bin"))
                soft.cpu().numpy().astype(np.complex64).view(np.float32).tofile(
                    os.path.join(ddir, "soft_symbols.f32"))
                pipe.write_diagnostics(os.path.join(ddir, "rx_diagnostics.jsonl"))
                write_adc_raw(os.path.join(ddir, "adc_stream.raw"),
                              AdcCodes(codes.cpu().numpy(), half, pipe_cfg.adc_rate_hz))
        except (SyncError, SyncFailure) as exc:
            point["status"] = "failed"
            point["reason"] = str(exc)
        points.append(point)
    report = {"schema_version": REPORT_SCHEMA_VERSION, "config": c, "points": points}
    if output_dir:
        os.makedirs(output_dir, exist_ok=True)
        with open(os.path.join(output_dir, "report.json"), "w") as f:
            json.dump(report, f, indent=2, sort_keys=True, default=float)
    return report


def _kkmodem():
    """The reference package (installed in baseline/_ref by
    tools/install_reference.py, or importable otherwise)."""
    import importlib
    import importlib.util
    import os
    import sys

    if importlib.util.find_spec("kkmodem") is None:
        ref = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
        if os.path.isdir(os.path.join(ref, "kkmodem")):
            os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/kkb200_numba_cache")
            sys.path.append(ref)
    try:
        return importlib.import_module("kkmodem.harness.sweep"), importlib.import_module("kkmodem.harness.config")
    except ImportError as exc:
        raise ParameterError("run_sweep drives the reference's own sweep driver: kkmodem must be importable "
                             "(tools/install_reference.py installs it into baseline/_ref)") from exc


def _run_single_nonlinear(c: dict, output_dir, save_captures) -> dict:
    """run_single for a nonlinear link: the split-step fiber is a whole-
    capture recurrence (channel.py ssfm_span :124-158 over the full signal,
    not chunkable like capgen's linear overlap-save), so the reference's own
    run_single (runner.py:140-196) runs with the backend switch installed --
    its ssfm_span spans and its receiver are this package's GPU ones
    (kkmodem_backend), transmitter / EDFAs / front end stay kkmodem's."""
    _kkmodem()
    import kkmodem.harness.config as kcfg
    import kkmodem.harness.runner as krun

    from . import kkmodem_backend
    kkmodem_backend.install()
    return krun.run_single(kcfg.ExperimentConfig.from_dict(c), output_dir, save_captures)


def run_sweep(cfg, output_dir: str | None = None) -> dict:
    """The reference's own sweep driver (kkmodem.harness.sweep.run_sweep,
    sweep.py:41-83: axis application, rows, per-distance argmax summary, the
    two CSV files) with every point's run_single on the GPU (this module's
    run_single: GPU capture generator + B200 receive + device metrics).
    `cfg`: the reference's ExperimentConfig or its dict layout."""
    sweep, config = _kkmodem()
    ec = cfg if isinstance(cfg, config.ExperimentConfig) else config.ExperimentConfig.from_dict(
        cfg.to_dict() if hasattr(cfg, "to_dict") else cfg)
    orig = sweep.run_single
    sweep.run_single = lambda point_cfg, *a, **k: run_single(point_cfg.to_dict())
    try:
        return sweep.run_sweep(ec, output_dir)
    finally:
        sweep.run_single = orig


def run_sustained(cfg, n_adc_samples: int, osnr_db: float | None = None, chunk_symbols: int = 1 << 16) -> dict:
    """Back-to-back contiguous streaming run with bounded memory
    (runner.py:290-348, same arguments and result keys).  The ADC stream is
    generated chunk by chunk on the GPU (capgen with the streaming front
    end's model: RRC shaping, carrier, optional OSNR noise loading, PD + ADC
    response, 12-bit quantizer; no dispersion, no phase noise, no OBPF),
    each chunk is fed to the receiver and its released decisions are scored
    against the transmitted PRBS bits; BER/Q over [startup + head guard,
    n - tail guard) and the windowed-Q trace, as in the reference."""
    import copy

    import torch

    from . import capgen

    c = copy.deepcopy(cfg.to_dict() if hasattr(cfg, "to_dict") else cfg)
    order = int(c["tx"]["constellation_order"])
    spec = make_constellation(order)
    k = spec.bits_per_symbol
    n_symbols = int(n_adc_samples) // 4
    c["tx"]["n_symbols"] = n_symbols
    c["link"].update(n_spans=1, span_length_km=0.0, ase_enabled=False, phase_noise_linewidth_hz=0.0)
    gp = capgen.GenParams.from_config(c)
    gp.osnr_db = osnr_db
    gp.obpf_enabled = False
    seed = int(np.random.SeedSequence(int(c.get("seed", 0))).generate_state(4)[0])   # hr:41-48 "link"
    gen = capgen.CaptureGenerator(gp, seed=seed)
    rx = c["rx"]
    n_ref = max(int(rx["sync_symbols"]), int(rx["startup_symbols"]))
    per = gen.period_bits
    ref_bits = np.take(per, np.arange(min(n_ref, n_symbols) * k) % len(per))
    ref = spec.points[capgen.map_symbols(ref_bits, order)]
    link = _namespace({"total_dispersion_ps_nm": 0.0, "center_wavelength_nm": c["link"]["center_wavelength_nm"]})
    pipe_cfg = make_pipeline_config(_namespace(c), link)
    pipe = RxPipeline(pipe_cfg, reference_symbols=ref)
    dev = pipe.dev
    labels, tx_idx = [], []
    for start in range(0, n_symbols, chunk_symbols):
        m = min(chunk_symbols, n_symbols - start)
        adc, idx, _ = gen.next_chunk(m)
        tx_idx.append(idx)
        pipe.feed(adc)
        lab, _, _ = pipe.drain_device(want_soft=False)
        labels.append(lab)
    pipe.feed(np.zeros(0), flush=True)
    lab, _, _ = pipe.drain_device(want_soft=False)
    labels.append(lab)
    lab = torch.cat(labels)[:n_symbols]
    txi = torch.from_numpy(np.concatenate(tx_idx)[:lab.shape[0]].astype(np.int64)).to(dev)
    # decisions -> bits on the device (training symbols are the reference's)
    dec_idx = torch.where(lab == 255, txi, lab.long())
    pl = torch.from_numpy(slicer_tables(order).point_label[:order].astype(np.int64)).to(dev)
    shifts = torch.arange(k - 1, -1, -1, device=dev)
    rx_bits = (pl[dec_idx][:, None] >> shifts) & 1
    tx_bits = (pl[txi][:, None] >> shifts) & 1
    flags = (rx_bits != tx_bits).to(torch.uint8).reshape(-1).cpu().numpy()
    error_flags = np.zeros(k * n_symbols, dtype=np.uint8)
    error_flags[:len(flags)] = flags
    m_cfg = c["metrics"]
    head = int(rx["startup_symbols"]) + int(m_cfg["head_guard_symbols"])
    stop_sym = n_symbols - int(m_cfg["tail_guard_symbols"])
    region = error_flags[head * k:stop_sym * k]
    n_errors = int(np.sum(region))
    ber = n_errors / len(region)
    series = windowed_q(region, float(c["tx"]["baud_hz"]) * k, float(m_cfg["windowed_q_window_s"]))
    qs = [q for _, q in series]
    return {
        "n_symbols": int(stop_sym - head),
        "n_bits": int(len(region)),
        "n_errors": n_errors,
        "ber": ber,
        "q_db": q_from_ber(ber) if ber > 0 else np.inf,
        "diverged": pipe.diverged,
        "windowed_q": series,
        "windowed_q_std_db": float(np.std(qs)) if len(qs) > 1 else 0.0,
    }


def measure_point(dec, soft, bits, syms, cfg) -> dict:
    """BER/Q/EVM over the post-startup region (hr:104-137)."""
    spec = make_constellation(cfg.tx.constellation_order)
    k = spec.bits_per_symbol
    head = cfg.rx.startup_symbols + cfg.metrics.head_guard_symbols
    stop = min(len(dec), len(syms)) - cfg.metrics.tail_guard_symbols
    if stop - head < 1000:
        raise SyncFailure("too few symbols beyond the startup region")
    rx_bits, _ = demap(dec[head:stop], spec)
    offset, a_rx, a_tx = frame_sync(rx_bits, bits)
    errors = a_rx != a_tx
    n_bits, n_err = len(errors), int(np.sum(errors))
    ber = n_err / n_bits
    point = {"ber": ber, "q_db": q_from_ber(ber), "evm_pct": evm(soft[head:stop], syms[head:stop]),
             "n_bits": n_bits, "n_errors": n_err, "sync_offset": int(offset)}
    bit_rate = cfg.tx.baud_hz * k
    win = cfg.metrics.windowed_q_window_s
    point["windowed_q"] = ([[float(t), float(q)] for t, q in windowed_q(errors, bit_rate, win)]
                           if n_bits >= int(win * bit_rate) else [])
    return point


def receive_batch(items, device=None, max_concurrency: int | None = None):
    """Batched multi-stream receive (sweeps): independent
    streams -- (cfg, adc, reference_symbols) each, adc a numpy / CUDA array,
    AdcCodes or AdcPacked12 -- whose front ends run as ONE set of launches
    (rxdsp.feed_batch: one K1 launch and one K2 launch per specialisation for
    all streams), syncs all enqueued before any is awaited, then every
    stream's DDLMS frames.  Returns, in order, (labels uint8, soft complex64)
    CUDA tensors per stream (on the caller's current stream) and the
    pipelines.  (max_concurrency: accepted for compatibility, unused.)"""
    import torch

    from .rxdsp import feed_batch

    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    pipes = [RxPipeline(cfg, reference_symbols=ref, device=dev) for cfg, _, ref in items]
    # one input format per launch: group the streams by it
    groups: dict = {}
    for i, (_, adc, _) in enumerate(items):
        key = type(adc).__name__ + (str(getattr(adc, "dtype", "")) if hasattr(adc, "dtype") else "")
        groups.setdefault(key, []).append(i)
    for idx in groups.values():
        feed_batch([pipes[i] for i in idx], [items[i][1] for i in idx], ddlms=False)
    # the DDLMS frames (independent recurrences): host-driven loops -- small
    # frames pay more for a CUDA-graph instantiation (~0.6 ms, allocating
    # device memory) than for the loop's readbacks (measured on the 11
    # goldens: 22.9 ms batched vs 33.6 ms with graphs; worker threads per
    # stream did not beat it: 32 ms)
    res = []
    for p in pipes:
        p._graph_loop = False
        t0 = p._ev()
        p._run_ddlms(True)
        p._events.append(("ddlms", t0, p._ev()))
        p._flushed = True
        lab, soft, _ = p.drain_device()
        res.append((lab, soft, p))
    return res


def frame_sync_device(rx_bits, tx_bits, min_peak_ratio: float = 3.0):
    """GPU frame_sync (metrics.py:69-112 semantics): bipolar cross-correlation
    of the received and transmitted bit streams (uint8 CUDA tensors) over all
    lags by kk_bit_xcorr (the repo's float64 Stockham FFT, rounded to the
    exact integer correlation), peak-to-sidelobe test excluding +-2 lags,
    linear correlation -- or circular when the lengths are equal.  Returns
    (lag, aligned rx bits, aligned tx bits) as device views."""
    import torch

    n_rx, n_tx = int(rx_bits.shape[0]), int(tx_bits.shape[0])
    if n_tx < (1 << 14):
        raise ParameterError("reference must be at least 2^14 bits")
    if n_rx < 64:
        raise SyncFailure("received stream too short")
    dev = rx_bits.device
    circular = int(n_rx == n_tx)
    rx_bits = rx_bits.contiguous()
    tx_bits = tx_bits.contiguous()
    nws = int(_lib.load().kk_bit_xcorr_workspace_bytes(n_rx, n_tx, circular))
    if nws == 0:
        raise ParameterError("bit streams too long for frame sync (correlation length > 2^31)")
    ws = torch.empty(nws, dtype=torch.uint8, device=dev)
    out = torch.empty(3, dtype=torch.int64, device=dev)
    _lib.call("kk_bit_xcorr", rx_bits.data_ptr(), n_rx, tx_bits.data_ptr(), n_tx, circular, ws.data_ptr(), nws,
              out.data_ptr(), torch.cuda.current_stream(dev).cuda_stream)
    k, peak, side = (int(v) for v in out.cpu())
    del ws
    ratio = peak / (side + 1e-30)
    if circular:
        if ratio < min_peak_ratio:
            raise SyncFailure(f"no circular correlation peak (ratio {ratio:.2f})")
        return k, torch.roll(rx_bits, -k), tx_bits
    if ratio < min_peak_ratio:
        raise SyncFailure(f"no correlation peak (ratio {ratio:.2f})")
    lag = (n_tx - 1) - k
    if lag >= 0:
        n = min(n_rx, n_tx - lag)
        return lag, rx_bits[:n], tx_bits[lag:lag + n]
    n = min(n_rx + lag, n_tx)
    return lag, rx_bits[-lag:-lag + n], tx_bits[:n]


def measure_point_device(labels, soft, bits, syms, cfg) -> dict:
    """measure_point (hr:104-137) with the decisions left on the GPU: labels
    (uint8 point indices) and soft (complex64) CUDA tensors, bits / syms the
    transmitted bits and symbols (host).  Labels -> bits (kk_label_bits),
    frame sync (kk_bit_xcorr), error and per-window counts
    (kk_bit_error_windows) and the EVM sums (kk_evm_sums) all run in the
    repo's kernels; only scalars and the window counts come back."""
    import torch

    spec = make_constellation(cfg.tx.constellation_order)
    k = spec.bits_per_symbol
    dev = labels.device
    st = torch.cuda.current_stream(dev).cuda_stream
    head = cfg.rx.startup_symbols + cfg.metrics.head_guard_symbols
    stop = min(int(labels.shape[0]), len(syms)) - cfg.metrics.tail_guard_symbols
    if stop - head < 1000:
        raise SyncFailure("too few symbols beyond the startup region")
    pl = np.ascontiguousarray(slicer_tables(spec.order).point_label, dtype=np.uint8)
    lab = labels[head:stop].contiguous()
    rx_bits = torch.empty(int(lab.shape[0]) * k, dtype=torch.uint8, device=dev)
    _lib.call("kk_label_bits", lab.data_ptr(), int(lab.shape[0]), pl.ctypes.data, spec.order, k,
              rx_bits.data_ptr(), st)
    tx_bits = torch.from_numpy(np.ascontiguousarray(bits, dtype=np.uint8)).to(dev)
    offset, a_rx, a_tx = frame_sync_device(rx_bits, tx_bits)
    a_rx, a_tx = a_rx.contiguous(), a_tx.contiguous()
    n_bits = int(a_rx.shape[0])
    bit_rate = cfg.tx.baud_hz * k
    win = cfg.metrics.windowed_q_window_s
    bpw = int(round(win * bit_rate))
    n_win = n_bits // bpw if (n_bits >= int(win * bit_rate) and bpw >= 1) else 0
    counts = torch.zeros(1 + max(n_win, 1), dtype=torch.int64, device=dev)
    _lib.call("kk_bit_error_windows", a_rx.data_ptr(), a_tx.data_ptr(), n_bits, bpw if n_win else 0,
              counts.data_ptr(), counts[1:].data_ptr() if n_win else None, st)
    s = soft[head:stop].contiguous()
    r = torch.from_numpy(np.ascontiguousarray(syms[head:stop], dtype=np.complex128)).to(dev)
    sums = torch.zeros(2 + 1024, dtype=torch.float64, device=dev)
    _lib.call("kk_evm_sums", s.data_ptr(), r.data_ptr(), int(s.shape[0]), sums.data_ptr(), sums[2:].data_ptr(), st)
    c = counts.cpu().numpy()
    se, sr = (float(v) for v in sums[:2].cpu())
    n_err = int(c[0])
    ber = n_err / n_bits
    evm_pct = float(100.0 * np.sqrt((se / s.shape[0]) / (sr / s.shape[0])))
    point = {"ber": ber, "q_db": q_from_ber(ber), "evm_pct": evm_pct, "n_bits": n_bits, "n_errors": n_err,
             "sync_offset": int(offset)}
    if n_win:
        point["windowed_q"] = [[float(t), float(q)] for t, q in windowed_q_from_counts(c[1:1 + n_win], bpw, win)]
    else:
        point["windowed_q"] = []
    return point


def device_ber(labels, ref_idx, order: int, head: int, stop: int, tile_symbols: int = 0, seam_guard: int = 128,
               index0: int = 0):
    """BER of decided indices [head, stop) against transmitted indices on the
    GPU (kk_bit_errors), excluding `seam_guard` symbols before every tile
    seam of a tiled capture.  Returns device
    tensors (errors, symbols).  index0: absolute symbol index of labels[0]
    (sets the seam phase)."""
    lab = labels[head:stop]
    ref = ref_idx[head:stop]
    if tile_symbols > 0:
        return count_bit_errors(lab, ref, order, exclude_period=tile_symbols, exclude_len=seam_guard,
                                exclude_phase=index0 + head)[:2]
    return count_bit_errors(lab, ref, order)[:2]


def pack_labels_host(labels, sym0: int, train_idx, order: int, bits_host) -> int:
    """Decided labels (uint8 point indices, 255 = training symbol) -> the
    demapped bit stream packed MSB first (kk_pack_bits, np.packbits layout)
    -> pinned host memory `bits_host`, on the current stream.  Training
    labels take the transmitted index train_idx[sym0 + i] (device uint8).
    Returns the bytes copied."""
    import torch

    n = int(labels.numel())
    if n == 0:
        return 0
    tb = slicer_tables(order)
    k = int(np.log2(order))
    nb = (n * k + 7) // 8
    if nb > bits_host.numel():
        raise ParameterError(f"bits_host holds {bits_host.numel()} bytes, need {nb}")
    dev = labels.device
    packed = torch.empty(nb, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream(dev).cuda_stream
    n_train = int(train_idx.numel()) if train_idx is not None else 0
    _lib.call("kk_pack_bits", labels.data_ptr(), n, int(sym0), train_idx.data_ptr() if n_train else None, n_train,
              k, tb.point_label.ctypes.data, order, packed.data_ptr(), st)
    bits_host[:nb].copy_(packed, non_blocking=True)
    return nb


# stream priorities of a streaming receive (KK_FRONT_PRIO / KK_DDLMS_PRIO:
# lower = scheduled first)
_FRONT_PRIO = int(__import__("os").environ.get("KK_FRONT_PRIO", "0"))


def receive_host_stream(cfg, host_codes, half_lsb: float, reference_symbols, chunk_samples: int = 1 << 25,
                        bits_host=None, device=None, staging=None, trace=None, packed12_samples: int | None = None):
    """End-to-end receive of an int16 ADC stream in pinned HOST memory; the
    receiver's output -- the demapped bit stream, packed (np.packbits
    layout) -- lands in pinned host memory.

    Every chunk's host->device copy is queued up front on a side stream into
    one device staging buffer (HBM is plentiful; the copy engine then streams
    at the full PCIe rate however long the receiver blocks the host), the
    compute stream waits per chunk on its copy event, and the bits of every
    completed DDLMS frame go back on a third stream as they are released --
    both PCIe directions overlap the GPU work.  `staging` (optional) is a
    reusable int16 device buffer of >= n samples.  The DDLMS tail frames
    are aligned to the chunk ends (RxPipeline.expect(chunk_ends=...)).
    packed12_samples=n: host_codes is instead a pinned uint8 buffer of the
    packed 12-bit wire format (sigcore.AdcPacked12, 1.5 B/sample) holding n
    samples; it is unpacked inside K1's staging (staging: uint8).
    Returns (pipe, bits_host, n_symbols_decided).
    """
    import torch

    from .constellation import make_constellation, slicer_tables
    from .sigcore import AdcCodes

    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    caller = torch.cuda.current_stream(dev)
    comp = side_stream(dev, "front", _FRONT_PRIO)
    comp.wait_stream(caller)
    with torch.cuda.stream(comp):
        out = _receive_host_stream(cfg, host_codes, half_lsb, reference_symbols, chunk_samples, bits_host, dev,
                                   staging, trace, comp, packed12_samples)
    caller.wait_stream(comp)
    return out


def _stream_receiver(cfg, reference_symbols, n: int, chunk_samples: int, dev, chunk_ends=None,
                     stage_timing: bool = False):
    """Pipeline + output packing state of a streaming receive (shared by the
    pinned-host and raw-file ingest paths)."""
    import dataclasses

    import torch

    from .constellation import make_constellation, slicer_tables

    # DDLMS frames run asynchronously (worker thread + stream) so the front
    # end of later chunks overlaps them.
    # No stage-timing events: each one drains the front-end stream before its
    # timestamp (~1 ms per 2^30-sample stream); stage_seconds reports zeros.
    gpu = dataclasses.replace(cfg.gpu, ddlms_async=True, stage_timing=stage_timing)
    cfg = dataclasses.replace(cfg, gpu=gpu)
    pipe = RxPipeline(cfg, reference_symbols=reference_symbols, device=dev)
    pipe.expect(n, chunk_samples, chunk_ends=chunk_ends)
    order = cfg.constellation_order
    st = {"cfg": cfg, "pipe": pipe, "order": order, "k": make_constellation(order).bits_per_symbol,
          "tb": slicer_tables(order), "train_idx": None, "n_train": 0, "n_out": 0, "b_out": 0}
    if reference_symbols is not None:
        ref = np.asarray(reference_symbols, np.complex128)[:cfg.ddlms.startup_symbols]
        pts = make_constellation(order).points
        ti = np.argmin(np.abs(ref[:, None] - pts[None, :]), axis=1).astype(np.uint8)
        st["train_idx"] = _upload(ti, dev)
        st["n_train"] = len(ti)
    return st


def _bits_capacity(cfg, n: int, k: int) -> int:
    """Upper bound of the packed output bytes of an n-sample stream: the flush
    zero-pads the KK and static hops, so up to (n + both FFT sizes) / 4
    symbols are decided."""
    n_sym = (n + cfg.static_plan.fft_size + cfg.kk_plan.fft_size) // 4 + 16
    return (n_sym * k + 7) // 8 + 8


def _drain_bits(st, bits_host, d2h, dev, max_frames=None, final: bool = False):
    """Finished frames -> packed bits -> pinned host, on the d2h stream (the
    other DMA direction), off the compute stream.  Whole groups of 8 symbols
    (k whole bytes) are packed; the remainder is carried to the next call so
    the byte stream is continuous whatever the frame sizes (final=True packs
    it)."""
    import torch

    pipe, k = st["pipe"], st["k"]
    lab, soft, _ = pipe.drain_device(wait_stream=d2h, want_soft=False, max_frames=max_frames)
    if lab.numel():
        lab.record_stream(d2h)
        soft.record_stream(d2h)
    carry = st.get("carry")
    if carry is not None and carry.numel():
        with torch.cuda.stream(d2h):
            lab = torch.cat([carry, lab]) if lab.numel() else carry
    n = int(lab.numel())
    n_pack = n if final else (n // 8) * 8
    st["carry"] = lab[n_pack:] if n_pack < n else None
    if n_pack == 0:
        return
    nb = (n_pack * k + 7) // 8
    ti = st["train_idx"]
    with torch.cuda.stream(d2h):
        packed = torch.empty(nb, dtype=torch.uint8, device=dev)
        _lib.call("kk_pack_bits", lab.data_ptr(), n_pack, st["n_out"],
                  ti.data_ptr() if ti is not None else None, st["n_train"], k,
                  st["tb"].point_label.ctypes.data, st["order"], packed.data_ptr(), d2h.cuda_stream)
        if st["b_out"] + nb > bits_host.numel():
            raise ParameterError(f"bits_host holds {bits_host.numel()} bytes, the stream needs more "
                                 f"(>= {st['b_out'] + nb})")
        bits_host[st["b_out"]:st["b_out"] + nb].copy_(packed, non_blocking=True)
    st["n_out"] += n_pack
    st["b_out"] += nb


def _receive_host_stream(cfg, host_codes, half_lsb, reference_symbols, chunk_samples, bits_host, dev, staging,
                         trace, comp, packed12_samples=None):
    import torch

    from .sigcore import AdcCodes, AdcPacked12

    p12 = packed12_samples is not None
    n = int(packed12_samples) if p12 else int(host_codes.shape[0])
    if p12 and (n % 2 or chunk_samples % 2):
        raise ParameterError("packed 12-bit streams and chunks hold even sample counts")

    def span(a, b):   # element range of samples [a, b) in the host / staging buffers
        return (3 * a // 2, 3 * b // 2) if p12 else (a, b)

    copy = side_stream(dev, "h2d")
    d2h = side_stream(dev, "d2h")
    n_el = span(0, n)[1]
    if staging is None or staging.numel() < n_el or (staging.dtype == torch.uint8) != p12:
        staging = torch.empty(n_el, dtype=torch.uint8 if p12 else torch.int16, device=dev)
    # (feeding the last chunk in smaller pieces was measured slower: the
    # DDLMS tail frames then form a longer chain of ~0.5 ms frame latencies)
    starts = list(range(0, n, chunk_samples))
    sizes = [b - a for a, b in zip(starts, starts[1:] + [n])]
    ready = [torch.cuda.Event(enable_timing=trace is not None) for _ in starts]
    copy.wait_stream(comp)          # the staging buffer's previous readers
    if trace is not None:
        import time

        ev0 = torch.cuda.Event(enable_timing=True)
        ev0.record(copy)
        trace.append(("copy_start", time.perf_counter(), ev0))

    def queue_copies(lo, hi):
        with torch.cuda.stream(copy):
            for i in range(lo, hi):
                e0, e1 = span(starts[i], starts[i] + sizes[i])
                staging[e0:e1].copy_(host_codes[e0:e1], non_blocking=True)
                ready[i].record(copy)

    # Every chunk's copy is queued first; the pipeline's set-up overlaps
    # them.  Its table uploads travel as kernel parameters (kk_upload): a DMA
    # copy issued now would wait for the whole queued stream on the
    # host->device copy engine.
    if bits_host is None:   # (pinned allocation before the copies are queued)
        k = make_constellation(cfg.constellation_order).bits_per_symbol
        bits_host = torch.empty(_bits_capacity(cfg, n, k), dtype=torch.uint8, pin_memory=True)
    queue_copies(0, len(starts))
    st = _stream_receiver(cfg, reference_symbols, n, chunk_samples, dev, chunk_ends=[a + m for a, m in
                                                                                   zip(starts, sizes)])
    pipe, cfg = st["pipe"], st["cfg"]
    for i, a in enumerate(starts):
        m = sizes[i]
        comp.wait_event(ready[i])
        if p12:
            e0, e1 = span(a, a + m)
            chunk = AdcPacked12(staging[e0:e1], half_lsb, m, cfg.adc_rate_hz)
        else:
            chunk = AdcCodes(staging[a:a + m], half_lsb, cfg.adc_rate_hz)
        pipe.feed(chunk, flush=i == len(starts) - 1)
        if trace is not None:
            import time

            ev = torch.cuda.Event(enable_timing=True)
            ev.record(comp)
            trace.append((i, time.perf_counter(), ready[i], ev, len(pipe._jobs)))
        # after the last chunk: ship each remaining frame as soon as it is
        # solved (its transfer overlaps the next frames' solves)
        while True:
            _drain_bits(st, bits_host, d2h, dev, max_frames=1 if i == len(starts) - 1 else None)
            if trace is not None:
                ev2 = torch.cuda.Event(enable_timing=True)
                ev2.record(d2h)
                trace.append(("d2h", time.perf_counter(), ev2))
            if i < len(starts) - 1 or not pipe.frames_pending:
                break
    _drain_bits(st, bits_host, d2h, dev, final=True)      # the last < 8 symbols
    comp.wait_stream(d2h)
    return pipe, bits_host, st["n_out"]


def receive_raw_file(cfg, path: str, reference_symbols, chunk_samples: int = 1 << 25, device=None,
                     n_buffers: int = 3):
    """Real-time ingest of the reference's int16 wire format (raw little-
    endian samples + JSON sidecar, sigcore.py:357-398): a reader thread
    reads the file chunk by chunk straight into pinned host buffers (ring of
    n_buffers), each is copied to the device on a side stream as soon as it
    is full and the receiver consumes it; disk/page-cache reads, PCIe copies
    and GPU work all overlap.  Returns (pipe, packed output bits (pinned
    host tensor), n_symbols_decided)."""
    import json
    import queue
    import threading

    import torch

    from .sigcore import AdcCodes, ParameterError

    with open(path + ".json") as f:
        meta = json.load(f)
    if meta.get("kind") != "int16":
        raise ParameterError("receive_raw_file: only int16 wire-format streams are supported")
    half_lsb = 1.0 / float(meta["scale"])
    n = int(meta["length"])
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    caller = torch.cuda.current_stream(dev)
    comp = side_stream(dev, "front", _FRONT_PRIO)
    copy = side_stream(dev, "h2d")
    d2h = side_stream(dev, "d2h")
    comp.wait_stream(caller)
    pins = [torch.empty(chunk_samples, dtype=torch.int16).pin_memory() for _ in range(n_buffers)]
    free_q, full_q = queue.Queue(), queue.Queue()
    for i in range(n_buffers):
        free_q.put((i, None))
    starts = list(range(0, n, chunk_samples))
    err = []

    def reader():
        try:
            with open(path, "rb") as f:
                for a in starts:
                    m = min(chunk_samples, n - a)
                    i, ev = free_q.get()
                    if ev is not None:
                        ev.synchronize()          # its previous H2D copy has finished
                    view = pins[i].numpy()[:m]
                    got = f.readinto(memoryview(view).cast("B"))
                    if got != 2 * m:
                        raise ParameterError(f"{path}: short read ({got} of {2 * m} bytes)")
                    full_q.put((i, m))
        except BaseException as exc:   # surfaced on the caller thread
            err.append(exc)
            full_q.put(None)

    th = threading.Thread(target=reader, daemon=True)
    with torch.cuda.stream(comp):
        st = _stream_receiver(cfg, reference_symbols, n, chunk_samples, dev)
        pipe, cfg = st["pipe"], st["cfg"]
        staging = torch.empty(n, dtype=torch.int16, device=dev)
        bits_host = torch.empty(_bits_capacity(cfg, n, st["k"]), dtype=torch.uint8, pin_memory=True)
        copy.wait_stream(comp)
        th.start()
        for ci, a in enumerate(starts):
            item = full_q.get()
            if item is None:
                raise err[0]
            i, m = item
            ready = torch.cuda.Event()
            with torch.cuda.stream(copy):
                staging[a:a + m].copy_(pins[i][:m], non_blocking=True)
                ready.record(copy)
            free_q.put((i, ready))
            comp.wait_event(ready)
            last = ci == len(starts) - 1
            pipe.feed(AdcCodes(staging[a:a + m], half_lsb, cfg.adc_rate_hz), flush=last)
            _drain_bits(st, bits_host, d2h, dev, max_frames=1 if last else None)
            while last and pipe.frames_pending:
                _drain_bits(st, bits_host, d2h, dev, max_frames=1)
            if last:
                _drain_bits(st, bits_host, d2h, dev, final=True)
        comp.wait_stream(d2h)
    th.join()
    if err:
        raise err[0]
    caller.wait_stream(comp)
    return pipe, bits_host, st["n_out"]
