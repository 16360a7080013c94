"""Golden vectors for the fiber span: run the REAL reference
kkmodem.channel.ssfm_span (channel.py:124-158) on seeded inputs and store
inputs, span parameters and outputs in tests/golden/channel_ssfm.npz.

    python tools/gen_golden_channel.py     # in the build container (needs kkmodem)
"""

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from gen_golden import REPO, kkmodem  # noqa: E402,F401  (imports the reference)

from kkmodem.channel import FiberSpan, ssfm_span  # noqa: E402
from kkmodem.sigcore import ComplexSignal  # noqa: E402

# (n, fs, length_km, loss_db_per_km, D, gamma, step_km, power_mw)
CASES = [
    (3000, 16e9, 100.0, 0.154, 20.0, 0.8, 10.0, 10.0),     # C8-like: non-power-of-two, 10 steps
    (4096, 16e9, 80.0, 0.2, 17.0, 1.3, 7.0, 20.0),         # power of two, rounded step count
    (1000, 32e9, 50.0, 0.0, 20.0, 0.0, None, 1.0),          # lossless, linear (default 1 km steps)
    (1 << 14, 16e9, 100.0, 0.154, 20.0, 0.8, 25.0, 50.0),  # strong nonlinearity
]


def main():
    out = {}
    for i, (n, fs, L, loss, D, g, step, p) in enumerate(CASES):
        rng = np.random.default_rng(100 + i)
        x = np.sqrt(p / 2) * (rng.standard_normal(n) + 1j * rng.standard_normal(n))
        span = FiberSpan(length_km=L, loss_db_per_km=loss, dispersion_ps_nm_km=D, gamma_per_w_km=g)
        y = ssfm_span(ComplexSignal(x, fs), span, step).samples
        out[f"x{i}"] = x
        out[f"y{i}"] = y
        out[f"p{i}"] = np.array([n, fs, L, loss, D, g, np.nan if step is None else step, p])
    path = os.path.join(REPO, "tests", "golden", "channel_ssfm.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, {k: v.shape for k, v in out.items() if k.startswith("y")})


if __name__ == "__main__":
    main()
