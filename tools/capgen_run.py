"""Generate a physical (non-tiled) 10,000 km QPSK capture on the GPU with
capgen, receive it, and report generation time, BER/EVM against the
reference capture's point."""
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from types import SimpleNamespace  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2108_07001_b200 import capgen, rxdsp  # noqa: E402
from paper_2108_07001_b200.captures import load_capture  # noqa: E402
from paper_2108_07001_b200.constellation import make_constellation  # noqa: E402
from paper_2108_07001_b200.harness import measure_point_device  # noqa: E402
from paper_2108_07001_b200.sigcore import AdcCodes  # noqa: E402

log2sym = int(sys.argv[1]) if len(sys.argv) > 1 else 22
cap = load_capture("c4_qpsk_10000km_cspr10")
c = cap.meta["config"]
n = 1 << log2sym
g = capgen.CaptureGenerator(capgen.GenParams.from_config(c), seed=7)
torch.cuda.synchronize()
t = time.perf_counter()
codes, half, idx, bits = g.generate(n, chunk_symbols=1 << 20)
torch.cuda.synchronize()
tg = time.perf_counter() - t
print(f"generated {n} symbols = {codes.numel()} ADC samples in {tg:.2f} s ({codes.numel() / tg / 1e9:.3f} GSa/s)")
pts = make_constellation(4).points
pipe = rxdsp.RxPipeline(cap.pipeline_config(), reference_symbols=pts[idx[:20000]])
t = time.perf_counter()
pipe.feed(AdcCodes(codes, half, 4e9))
pipe.feed(np.zeros(0), flush=True)
lab, soft, _ = pipe.drain_device()
torch.cuda.synchronize()
print(f"received in {time.perf_counter() - t:.3f} s, sync offset {pipe.sync_offset}")
cfgx = SimpleNamespace(tx=SimpleNamespace(constellation_order=4, baud_hz=1e9),
                       rx=SimpleNamespace(startup_symbols=c["rx"]["startup_symbols"]),
                       metrics=SimpleNamespace(head_guard_symbols=2048, tail_guard_symbols=4096,
                                               windowed_q_window_s=0.021))
if n <= (1 << 22):
    pt = measure_point_device(lab, soft, bits, pts[idx], cfgx)
    print({k: v for k, v in pt.items() if k != "windowed_q"})
else:
    # beyond one PRBS-23 period frame_sync is ambiguous (periodic reference):
    # count against the known alignment (decision k <-> transmitted symbol k)
    from paper_2108_07001_b200.harness import device_ber
    ref_idx = torch.from_numpy(idx[:lab.shape[0]]).to(lab.device)
    head = c["rx"]["startup_symbols"] + 2048
    e, nb = device_ber(lab, ref_idx, 4, head, lab.shape[0] - 4096)
    print({"ber": int(e) / (2 * int(nb)), "n_errors": int(e), "n_bits": 2 * int(nb)})
print("reference capture point (2^16 symbols):", cap.meta["point"])
