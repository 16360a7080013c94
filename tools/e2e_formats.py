"""End-to-end streaming receive (pinned host int16 -> packed bits) of GPU-generated 16-/64-QAM captures (2^28 samples): wall time per stream and DDLMS iterations per frame."""
import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2108_07001_b200 import capgen
from paper_2108_07001_b200.captures import load_capture
from paper_2108_07001_b200.constellation import make_constellation
from paper_2108_07001_b200.harness import receive_host_stream
for name in ["c3_64qam_1600km_rel-20", "c2_16qam_5600km_rel-20"]:
    cap = load_capture(name); c = cap.meta["config"]
    gen = capgen.CaptureGenerator(capgen.GenParams.from_config(c), seed=7)
    codes, half, idx, _ = gen.generate(1 << 26, chunk_symbols=1 << 20)
    host = codes.cpu().pin_memory(); del codes
    pts = make_constellation(cap.order).points
    cfg = cap.pipeline_config(ddlms_frame_symbols=1 << 26)
    ref = pts[idx[:10000]]
    for rep in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        pipe, bits, n = receive_host_stream(cfg, host, half, ref)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
        pipe.release_buffers()
        print(name, f"e2e {n / dt / 1e9:.3f} GBaud ({dt*1e3:.1f} ms)", [s.get("iterations") for s in pipe.ddlms_stats], flush=True)
