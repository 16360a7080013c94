"""Golden fixture for harness.run_sustained: the reference's own
run_sustained (runner.py:290-348) on the configuration of its test
(test_harness.py:197-206: 16-QAM back-to-back, 8000 startup symbols, 0.2 ms
Q windows, 2^21 ADC samples, OSNR 22 dB), run HERE from /root/reference.
Writes tests/golden/harness/sustained_16qam_osnr22.json (config + result)."""
import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
from kkmodem.harness.config import preset  # noqa: E402
from kkmodem.harness.runner import run_sustained  # noqa: E402

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cfg = preset("ci")
cfg.tx.n_symbols = 1 << 16
cfg.tx.cspr_db = 12.0
cfg.link.n_spans = 1
cfg.link.span_length_km = 0.0
cfg.link.ase_enabled = False
cfg.link.phase_noise_linewidth_hz = 0.0
cfg.link.monitor_every_n_spans = 1
cfg.tx.constellation_order = 16
cfg.rx.startup_symbols = 8000
cfg.metrics.windowed_q_window_s = 2e-4
n, osnr = 1 << 21, 22.0
r = run_sustained(cfg, n_adc_samples=n, osnr_db=osnr)
out = {"generator": "tools/gen_golden_sustained.py (reference kkmodem run_sustained)",
       "config": cfg.to_dict(), "n_adc_samples": n, "osnr_db": osnr,
       "result": {k: (v if k != "windowed_q" else [[float(a), float(b)] for a, b in v])
                  for k, v in r.items()}}
with open(os.path.join(REPO, "tests", "golden", "harness", "sustained_16qam_osnr22.json"), "w") as f:
    json.dump(out, f, indent=1, default=float)
print(out["result"])
