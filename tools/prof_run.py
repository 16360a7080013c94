"""Short device-resident receive for profiling (ncu): one 2^N-sample feed of
the tiled 10,000 km QPSK capture through RxPipeline (all kernels launch)."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import torch  # noqa: E402

from paper_2108_07001_b200 import rxdsp  # noqa: E402
from paper_2108_07001_b200.captures import load_capture, tile  # noqa: E402
from paper_2108_07001_b200.sigcore import AdcCodes  # noqa: E402

log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cap = load_capture("c5_qpsk_10000km_tile")
codes, _ = tile(cap, 1 << log2n)
gpu_kw = {}
if os.environ.get("KK_FRAME_LOG2"):
    gpu_kw["ddlms_frame_symbols"] = 1 << int(os.environ["KK_FRAME_LOG2"])
cfg = cap.pipeline_config(**gpu_kw)
ref = cap.symbols()[:10000]
dev = torch.device("cuda", 0)
cd = torch.from_numpy(codes).to(dev)
for i in range(reps):
    pipe = rxdsp.RxPipeline(cfg, reference_symbols=ref)
    pipe.feed(AdcCodes(cd, cap.half_lsb), flush=True)
    lab, soft, meta = pipe.drain_device()
    torch.cuda.synchronize()
    print(i, lab.shape[0], pipe.stage_seconds, pipe.ddlms_stats)
