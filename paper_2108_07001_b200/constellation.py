"""Constellation tables (kkmodem.txdsp.make_constellation, txdsp.py:115-142)
plus the slicer descriptors the CUDA decision kernels use.

Point order and labels follow the reference exactly (QPSK table txdsp.py:36-41,
two-ring 8-QAM txdsp.py:44-46, per-axis Gray square QAM txdsp.py:102-112,
quasi-Gray 32-cross txdsp.py:52-63), so point indices are interchangeable
with the reference's.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from .sigcore import ParameterError

_QPSK = {0b00: 1 + 1j, 0b01: -1 + 1j, 0b11: -1 - 1j, 0b10: 1 - 1j}
_CROSS32 = {
    (-5, -3): 0b11001, (-5, -1): 0b11101, (-5, 1): 0b11111, (-5, 3): 0b11011,
    (-3, -5): 0b11010, (-3, -3): 0b11000, (-3, -1): 0b01101, (-3, 1): 0b01111,
    (-3, 3): 0b01011, (-3, 5): 0b01001, (-1, -5): 0b11110, (-1, -3): 0b11100,
    (-1, -1): 0b01100, (-1, 1): 0b01110, (-1, 3): 0b01010, (-1, 5): 0b01000,
    (1, -5): 0b10110, (1, -3): 0b10100, (1, -1): 0b00100, (1, 1): 0b00110,
    (1, 3): 0b00010, (1, 5): 0b00000, (3, -5): 0b10010, (3, -3): 0b10000,
    (3, -1): 0b00101, (3, 1): 0b00111, (3, 3): 0b00011, (3, 5): 0b00001,
    (5, -3): 0b10001, (5, -1): 0b10101, (5, 1): 0b10111, (5, 3): 0b10011,
}


@dataclass
class ConstellationSpec:
    order: int
    points: np.ndarray
    labels: np.ndarray

    @property
    def bits_per_symbol(self) -> int:
        return int(np.log2(self.order))

    @property
    def max_radius(self) -> float:
        return float(np.max(np.abs(self.points)))

    def label_to_index(self) -> np.ndarray:
        inv = np.empty(self.order, dtype=np.int64)
        inv[self.labels] = np.arange(self.order)
        return inv


@lru_cache(maxsize=None)
def make_constellation(order: int) -> ConstellationSpec:
    if order == 4:
        labs = np.array(sorted(_QPSK))
        pts = np.array([_QPSK[k] for k in labs])
    elif order == 8:
        ratio = (1.0 + np.sqrt(3.0)) / np.sqrt(2.0)
        gray4 = (0b00, 0b01, 0b11, 0b10)
        pts, labs = [], []
        for ring, (rad, degs) in enumerate(((1.0, (45, 135, 225, 315)), (ratio, (0, 90, 180, 270)))):
            for q, ang in enumerate(np.deg2rad(degs)):
                pts.append(rad * np.exp(1j * ang))
                labs.append((ring << 2) | gray4[q])
        pts, labs = np.array(pts), np.array(labs)
    elif order in (16, 64):
        m = int(np.sqrt(order))
        lv = np.arange(-(m - 1), m, 2, dtype=np.float64)
        kb = int(np.log2(m))
        gray = [i ^ (i >> 1) for i in range(m)]
        pts = np.array([lv[i] + 1j * lv[q] for i in range(m) for q in range(m)])
        labs = np.array([(gray[i] << kb) | gray[q] for i in range(m) for q in range(m)])
    elif order == 32:
        items = sorted(_CROSS32.items())
        pts = np.array([i + 1j * q for (i, q), _ in items])
        labs = np.array([lab for _, lab in items])
    else:
        raise ParameterError(f"unsupported constellation order {order}")
    pts = pts / np.sqrt(np.mean(np.abs(pts) ** 2))
    return ConstellationSpec(order, pts.astype(np.complex128), labs.astype(np.int64))


@dataclass
class SlicerTables:
    """Host arrays handed to the CUDA slicer (kk_ddlms_* entry points)."""

    order: int
    pts_ri: np.ndarray      # float32 [2*order] (re, im)
    grid: np.ndarray        # uint8 [m*m] (i_re*m + i_im) -> point index; empty: brute force
    grid_m: int
    norm: float             # level value = (2 i - (m-1)) / norm
    max_radius: float
    point_label: np.ndarray  # uint8 [64] point index -> bit label


@lru_cache(maxsize=None)
def slicer_tables(order: int) -> SlicerTables:
    spec = make_constellation(order)
    pts = spec.points
    pts_ri = np.empty(2 * order, dtype=np.float32)
    pts_ri[0::2] = pts.real
    pts_ri[1::2] = pts.imag
    m = int(round(np.sqrt(order)))
    grid = np.zeros(0, dtype=np.uint8)
    grid_m = 0
    norm = 1.0
    if m * m == order:
        # square grid: levels (2i-(m-1))/norm on both axes
        raw = np.arange(-(m - 1), m, 2, dtype=np.float64)
        norm_c = np.sqrt(np.mean(np.abs(raw[:, None] + 1j * raw[None, :]) ** 2))
        lv = raw / norm_c
        g = np.full(m * m, 255, dtype=np.uint8)
        ok = True
        for idx, p in enumerate(pts):
            ir = np.argmin(np.abs(lv - p.real))
            ii = np.argmin(np.abs(lv - p.imag))
            if abs(lv[ir] - p.real) > 1e-12 or abs(lv[ii] - p.imag) > 1e-12:
                ok = False
                break
            g[ir * m + ii] = idx
        if ok and np.all(g != 255):
            grid, grid_m, norm = g, m, float(norm_c)
    pl = np.zeros(64, dtype=np.uint8)
    pl[:order] = spec.labels.astype(np.uint8)
    return SlicerTables(order, pts_ri, grid, grid_m, norm, spec.max_radius, pl)
