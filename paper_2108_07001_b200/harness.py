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
from .constellation import make_constellation
from .metrics import SyncFailure, count_bit_errors, evm, frame_sync, q_from_ber, windowed_q
from .rxdsp import side_stream
from .rxdsp import (
    DdlmsConfig, GpuOptions, RxPipeline, RxPipelineConfig, compute_static_taps, demap, design_receive_taps,
)

from .sigcore import BlockPlan


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


def receive_host_stream(cfg, host_codes, half_lsb: float, reference_symbols, chunk_samples: int = 1 << 25,
                        bits_host=None, device=None, staging=None, trace=None):
    """End-to-end receive of an int16 ADC stream in pinned HOST memory; the
    receiver's output -- the demapped bit stream, packed (np.packbits
    layout) -- lands in pinned host memory.

    Every chunk's host->device copy is queued up front on a side stream into
    one device staging buffer (HBM is plentiful; the copy engine then streams
    at the full PCIe rate however long the receiver blocks the host), the
    compute stream waits per chunk on its copy event, and the bits of every
    completed DDLMS frame go back on a third stream as they are released --
    both PCIe directions overlap the GPU work.  `staging` (optional) is a
    reusable int16 device buffer of >= n samples.
    Returns (pipe, bits_host, n_symbols_decided).
    """
    import torch

    from .constellation import make_constellation, slicer_tables
    from .sigcore import AdcCodes

    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    caller = torch.cuda.current_stream(dev)
    comp = side_stream(dev, "front")
    comp.wait_stream(caller)
    with torch.cuda.stream(comp):
        out = _receive_host_stream(cfg, host_codes, half_lsb, reference_symbols, chunk_samples, bits_host, dev,
                                   staging, trace, comp)
    caller.wait_stream(comp)
    return out


def _receive_host_stream(cfg, host_codes, half_lsb, reference_symbols, chunk_samples, bits_host, dev, staging,
                         trace, comp):
    import torch

    from .constellation import make_constellation, slicer_tables
    from .sigcore import AdcCodes

    n = int(host_codes.shape[0])
    copy = side_stream(dev, "h2d")
    d2h = side_stream(dev, "d2h")
    if staging is None or staging.numel() < n:
        staging = torch.empty(n, dtype=torch.int16, device=dev)
    # the pipeline's own uploads go first: later small H2D copies would queue
    # behind the bulk transfers on the in-order host->device copy engine.
    # DDLMS frames run asynchronously (worker thread + stream) so the front
    # end of later chunks overlaps them.
    import dataclasses

    gpu = dataclasses.replace(cfg.gpu, ddlms_async=True)
    cfg = dataclasses.replace(cfg, gpu=gpu)
    pipe = RxPipeline(cfg, reference_symbols=reference_symbols, device=dev)
    pipe.expect(n, chunk_samples)
    order = cfg.constellation_order
    k = make_constellation(order).bits_per_symbol
    tb = slicer_tables(order)
    train_idx = None
    n_train = 0
    if reference_symbols is not None:
        ref = np.asarray(reference_symbols, np.complex128)[:cfg.ddlms.startup_symbols]
        pts = make_constellation(order).points
        ti = np.argmin(np.abs(ref[:, None] - pts[None, :]), axis=1).astype(np.uint8)
        train_idx = torch.from_numpy(ti).to(dev)
        n_train = len(ti)
    starts = list(range(0, n, chunk_samples))
    ready = [torch.cuda.Event() for _ in starts]
    copy.wait_stream(comp)          # the staging buffer's previous readers (and the uploads)
    with torch.cuda.stream(copy):
        for i, a in enumerate(starts):
            m = min(chunk_samples, n - a)
            staging[a:a + m].copy_(host_codes[a:a + m], non_blocking=True)
            ready[i].record(copy)
    if bits_host is None:
        bits_host = torch.empty((n // 4 + 8) * k // 8 + 8, dtype=torch.uint8, pin_memory=True)
    n_out = 0
    b_out = 0
    for i, a in enumerate(starts):
        m = min(chunk_samples, n - a)
        comp.wait_event(ready[i])
        pipe.feed(AdcCodes(staging[a:a + m], half_lsb, cfg.adc_rate_hz), flush=i == len(starts) - 1)
        if trace is not None:
            import time

            ev = torch.cuda.Event(enable_timing=True)
            ev.record(comp)
            trace.append((i, time.perf_counter(), ready[i], ev, len(pipe._jobs)))
        # finished frames, valid on the d2h stream: pack + device -> host there
        # (the other DMA direction), off the compute stream
        lab, soft, _ = pipe.drain_device(wait_stream=d2h)
        if lab.numel():
            nb = (lab.numel() * k + 7) // 8
            with torch.cuda.stream(d2h):
                packed = torch.empty(nb, dtype=torch.uint8, device=dev)
                _lib.call("kk_pack_bits", lab.data_ptr(), lab.numel(), n_out,
                          train_idx.data_ptr() if train_idx is not None else None, n_train, k,
                          tb.point_label.ctypes.data, order, packed.data_ptr(), d2h.cuda_stream)
                bits_host[b_out:b_out + nb].copy_(packed, non_blocking=True)
            lab.record_stream(d2h)
            soft.record_stream(d2h)
            n_out += lab.numel()
            b_out += nb
    comp.wait_stream(d2h)
    return pipe, bits_host, n_out
