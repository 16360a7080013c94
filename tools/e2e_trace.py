import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2108_07001_b200.captures import load_capture, tile
from paper_2108_07001_b200.harness import receive_host_stream
from paper_2108_07001_b200.sigcore import pack12
import dataclasses
cap = load_capture("c5_qpsk_10000km_tile")
cfg = cap.pipeline_config()
cfg = dataclasses.replace(cfg, gpu=dataclasses.replace(cfg.gpu, ddlms_frame_symbols=1 << int(os.environ.get("KK_E2E_FRAME_LOG2", "25")), ddlms_tail_min_symbols=1 << int(os.environ.get("KK_E2E_TAIL_LOG2", "25"))))
codes, _ = tile(cap, 1 << 30)
host = torch.from_numpy(pack12(codes)).pin_memory()
pts = cap.symbols()[:10000]
bits = torch.empty((1 << 30) // 4 * 2 // 8 + 65536, dtype=torch.uint8).pin_memory()
st = torch.empty(3 << 29, dtype=torch.uint8, device="cuda")
for i in range(5):
    torch.cuda.synchronize()
    t = time.perf_counter()
    pipe, bh, n = receive_host_stream(cfg, host, cap.half_lsb, pts, chunk_samples=1 << int(os.environ.get("KK_E2E_CHUNK_LOG2", "25")), bits_host=bits, staging=st, packed12_samples=1 << 30)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"e2e step {i}: {dt*1e3:.1f} ms  {n/dt/1e9:.3f} GBaud", [(s['nsym'], s.get('iterations'), s.get('mode')) for s in pipe.ddlms_stats], flush=True)
    pipe.release_buffers()
