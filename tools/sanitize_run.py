"""Small end-to-end receive for compute-sanitizer (memcheck / racecheck /
synccheck): the c4 golden capture through RxPipeline (K1, carrier, K2, sync,
DDLMS solver incl. training, scans, list passes) plus the packed-bit e2e path
(async DDLMS worker) and the capture generator."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2108_07001_b200 import rxdsp  # noqa: E402
from paper_2108_07001_b200.captures import load_capture  # noqa: E402
from paper_2108_07001_b200.harness import receive_host_stream  # noqa: E402

cap = load_capture("c4_qpsk_10000km_cspr10")
cfg = cap.pipeline_config(ddlms_frame_symbols=1 << 15)
pipe = rxdsp.RxPipeline(cfg, reference_symbols=cap.symbols())
pipe.feed(cap.adc)
dec, soft = pipe.finish()
print("decisions", len(dec))
_, bits, n = receive_host_stream(cfg, torch.from_numpy(cap.adc_h).pin_memory(), cap.half_lsb, cap.symbols(),
                                 chunk_samples=1 << 16)
torch.cuda.synchronize()
print("stream decisions", n)
