"""Captured ADC streams: the int16 wire format + transmitted symbols.

A capture is what the reference's own data path produces
(harness/runner.py:148-166: transmitter -> link -> photodiode -> 12-bit ADC),
stored as exact odd half-LSB int16 codes (value = code * lsb/2) plus the
transmitted symbols as constellation indices and the receive taps.
tools/gen_golden.py writes them under tests/golden/ from the real reference;
this module only reads them.  `tile` builds the long streaming workloads the
way bench_throughput does (runner.py:389-391 np.tile), with tiles of k*1000
ADC samples so the 0.516 GHz tone stays phase-continuous across seams.
"""

from __future__ import annotations

import json
import os
from dataclasses import dataclass

import numpy as np

from .sigcore import AdcCodes, BlockPlan, FirFilter

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")


@dataclass
class Capture:
    name: str
    meta: dict
    adc_h: np.ndarray        # int16 odd half-LSB codes
    half_lsb: float
    sym_idx: np.ndarray      # uint8 transmitted point indices
    taps: np.ndarray         # complex128 static receive taps @ adc_rate/2
    arrays: dict

    @property
    def order(self) -> int:
        return int(self.meta["order"])

    @property
    def adc(self) -> AdcCodes:
        return AdcCodes(self.adc_h, self.half_lsb, 4e9)

    def adc_float(self) -> np.ndarray:
        return self.adc_h.astype(np.float64) * self.half_lsb

    def symbols(self) -> np.ndarray:
        from .constellation import make_constellation
        return make_constellation(self.order).points[self.sym_idx]

    def pipeline_config(self, **gpu_kw):
        """RxPipelineConfig equal to make_pipeline_config's (runner.py:65-91)
        for the capture's experiment config."""
        from .rxdsp import DdlmsConfig, GpuOptions, RxPipelineConfig

        m = self.meta
        cfg = m["config"]
        return RxPipelineConfig(
            adc_rate_hz=cfg["frontend"]["adc_rate_hz"], baud_hz=cfg["tx"]["baud_hz"],
            tone_freq_hz=cfg["tx"]["tone_freq_hz"],
            kk_plan=BlockPlan(cfg["rx"]["kk_fft_size"], buffer_len=cfg["rx"]["buffer_len"]),
            static_plan=BlockPlan(cfg["rx"]["static_fft_size"], buffer_len=cfg["rx"]["buffer_len"]),
            static_taps=FirFilter(self.taps, cfg["frontend"]["adc_rate_hz"] / 2.0),
            carrier_removal=cfg["rx"]["carrier_removal"], carrier_segment_len=cfg["rx"]["carrier_segment_len"],
            ddlms=DdlmsConfig(mu=cfg["rx"]["mu"], startup_symbols=cfg["rx"]["startup_symbols"],
                              widely_linear=cfg["rx"]["widely_linear"]),
            constellation_order=cfg["tx"]["constellation_order"], sync_symbols=cfg["rx"]["sync_symbols"],
            sync_wait_samples=cfg["rx"]["sync_wait_samples"], gpu=GpuOptions(**gpu_kw))


def list_captures() -> list[str]:
    return sorted(f[:-5] for f in os.listdir(GOLDEN)
                  if f.endswith(".json") and os.path.exists(os.path.join(GOLDEN, f[:-5] + ".npz")))


def load_capture(name: str, directory: str = GOLDEN) -> Capture:
    with open(os.path.join(directory, f"{name}.json")) as f:
        meta = json.load(f)
    z = np.load(os.path.join(directory, f"{name}.npz"))
    arrays = {k: z[k] for k in z.files}
    return Capture(name=name, meta=meta, adc_h=arrays["adc_h"], half_lsb=meta["lsb"] / 2.0,
                   sym_idx=arrays["sym_idx"], taps=arrays["taps"], arrays=arrays)


def tile(cap: Capture, n_samples: int):
    """(int16 codes[n_samples], symbol indices[n_samples // 4]) tiled from
    the capture (runner.py:389-391 pattern)."""
    reps = -(-n_samples // len(cap.adc_h))
    codes = np.tile(cap.adc_h, reps)[:n_samples]
    syms = np.tile(cap.sym_idx, reps)[:n_samples // 4]
    return codes, syms
