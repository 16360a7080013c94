"""Device-resident receive of the 2^N-sample bench stream fed in chunks with
asynchronous DDLMS frames (the streaming schedule without the H2D leg): does
overlapping the frame chain with the front end of later chunks beat the
one-feed serial schedule?  argv: log2 samples, log2 chunk, log2 frame."""
import dataclasses
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import torch  # noqa: E402

from paper_2108_07001_b200 import rxdsp  # noqa: E402
from paper_2108_07001_b200.captures import load_capture, tile  # noqa: E402
from paper_2108_07001_b200.sigcore import AdcCodes  # noqa: E402

log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
chunk = 1 << int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 25
frame = 1 << int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 26
cap = load_capture("c5_qpsk_10000km_tile")
codes, _ = tile(cap, 1 << log2n)
dev = torch.device("cuda", 0)
cd = torch.from_numpy(codes).to(dev)
ref = cap.symbols()[:10000]
n = cd.shape[0]


def run(mode):
    if mode == "serial":
        cfg = cap.pipeline_config()
        pipe = rxdsp.RxPipeline(cfg, reference_symbols=ref, device=dev)
        pipe.feed(AdcCodes(cd, cap.half_lsb), flush=True)
        lab, _, _ = pipe.drain_device()
    else:
        cfg = cap.pipeline_config(ddlms_frame_symbols=frame)
        cfg = dataclasses.replace(cfg, gpu=dataclasses.replace(cfg.gpu, ddlms_async=True))
        pipe = rxdsp.RxPipeline(cfg, reference_symbols=ref, device=dev)
        starts = list(range(0, n, chunk))
        pipe.expect(n, chunk, chunk_ends=[min(a + chunk, n) for a in starts])
        labs = []
        for i, a in enumerate(starts):
            pipe.feed(AdcCodes(cd[a:a + chunk], cap.half_lsb), flush=i == len(starts) - 1)
            lab, _, _ = pipe.drain_device(want_soft=False)
            labs.append(lab)
        while pipe.frames_pending:
            lab, _, _ = pipe.drain_device(want_soft=False)
            labs.append(lab)
        lab = torch.cat(labs)
    return pipe, lab


for mode in ("serial", "async", "serial", "async", "serial", "async"):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    pipe, lab = run(mode)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{mode:7s}: {ms:7.2f} ms  {lab.numel() / ms / 1e6:6.3f} GBaud  symbols {lab.numel()}", flush=True)
    pipe.release_buffers()
