"""DDLMS block-size sweep on the bench workload (device-resident)."""
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import torch  # noqa: E402

from paper_2108_07001_b200 import rxdsp  # noqa: E402
from paper_2108_07001_b200.captures import load_capture, tile  # noqa: E402
from paper_2108_07001_b200.sigcore import AdcCodes  # noqa: E402

log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
cap = load_capture("c5_qpsk_10000km_tile")
codes, syms = tile(cap, 1 << log2n)
ref = cap.symbols()[:10000]
cd = torch.from_numpy(codes).cuda()
sym_idx = torch.from_numpy(syms).cuda()
base = None
for B in [int(b) for b in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["256", "512", "1024"])]:
    for rep in range(2):
        cfg = cap.pipeline_config(ddlms_block=B)
        pipe = rxdsp.RxPipeline(cfg, reference_symbols=ref)
        torch.cuda.synchronize()
        t = time.perf_counter()
        pipe.feed(AdcCodes(cd, cap.half_lsb), flush=True)
        lab, soft, meta = pipe.drain_device()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t
    st = pipe.stage_seconds
    if base is None:
        base = lab.clone()
    agree = float((lab == base).float().mean())
    print(f"B={B} wall={wall*1e3:.1f}ms ddlms={st['ddlms']/2*1e3:.2f}ms static={st['static']/2*1e3:.2f} kk={st['kk']/2*1e3:.2f}"
          f" agree_vs_first={agree:.7f} {pipe.ddlms_stats[-1]['per_iter']}", flush=True)
    pipe.release_buffers()
