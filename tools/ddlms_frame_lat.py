"""Latency of one DDLMS frame solve (kk_ddlms_solve) vs frame size and block
size B, on the bench capture's real equaliser input (front end run on a
tiled 10,000 km QPSK stream, frames deferred), frames after the training
section (the streaming tail case).  Prints device ms (events), host ms and
the iteration statistics."""
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2108_07001_b200 import _lib, rxdsp  # noqa: E402
from paper_2108_07001_b200.captures import load_capture, tile  # noqa: E402
from paper_2108_07001_b200.sigcore import AdcCodes  # noqa: E402

log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
sizes = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "20,21,22,23,24,25").split(",")]
blocks = [int(v) for v in (sys.argv[3] if len(sys.argv) > 3 else "64,128,256,512").split(",")]
cap = load_capture("c5_qpsk_10000km_tile")
codes, _ = tile(cap, 1 << log2n)
cfg = cap.pipeline_config(ddlms_frame_symbols=1 << 34)
dev = torch.device("cuda", 0)
pipe = rxdsp.RxPipeline(cfg, reference_symbols=cap.symbols()[:10000], device=dev)
AT_END = os.environ.get("KK_LAT_AT_END") == "1"     # frames ending at the flushed stream end
pipe.front_end(AdcCodes(torch.from_numpy(codes).to(dev), cap.half_lsb, cfg.adc_rate_hz), flush=AT_END)
pipe._run_ddlms(False)            # sync only (frames deferred: F is huge)
torch.cuda.synchronize()
k0 = 1 << 20                      # past the training section
total = (pipe._y2.end - pipe._drop - 4) // 2 + 1
tb = pipe._tables
d = cfg.ddlms
s = torch.cuda.current_stream(dev)
if os.environ.get("KK_LAT_PRIO"):
    s = torch.cuda.Stream(device=dev, priority=int(os.environ["KK_LAT_PRIO"]))
flush_buf = torch.empty(1 << 26, dtype=torch.float32, device=dev)
if os.environ.get("KK_LAT_HEAT") == "1":
    heat_codes = torch.from_numpy(codes).to(dev)
for lg in sizes:
    nsym = 1 << lg
    if AT_END:
        k0 = total - nsym
    for B in blocks:
        wsb = int(_lib.load().kk_ddlms_workspace_bytes(nsym, B))
        if os.environ.get("KK_LAT_BIG_WS"):
            wsb = max(wsb, int(_lib.load().kk_ddlms_workspace_bytes(1 << 26, 512)))
        ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
        lab = torch.empty(nsym, dtype=torch.uint8, device=dev)
        soft = torch.empty(nsym, dtype=torch.complex64, device=dev)
        dev_ms, host_ms = [], []
        for rep in range(4):
            Tin = np.ascontiguousarray(pipe._T_dev.cpu().numpy(), np.float32)
            Tout = np.zeros(16, np.float32)
            st = np.zeros(38, np.int64)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if os.environ.get("KK_LAT_FLUSH_L2") == "1":
                flush_buf.fill_(rep)      # evict L2 (256 MB > 126 MB)
            torch.cuda.synchronize()
            if os.environ.get("KK_LAT_HEAT") == "1":
                # ~40 ms of the receiver's own front end right before the solve
                # (is the frame slower on a GPU that just ran the full chain?)
                for _ in range(4):
                    heat = rxdsp.RxPipeline(cfg, reference_symbols=cap.symbols()[:10000], device=dev)
                    heat.front_end(AdcCodes(heat_codes, cap.half_lsb, cfg.adc_rate_hz), flush=False)
                    heat.release_buffers()
            else:
                torch.cuda.synchronize()
            h0 = time.perf_counter()
            e0.record(s)
            _lib.call("kk_ddlms_solve", pipe._y2.ptr(pipe._drop + 2 * k0), nsym, float(pipe._eq_scale), None, 0,
                      Tin.ctypes.data, tb.order, tb.pts_ri.ctypes.data, tb.grid.ctypes.data if tb.grid_m else None,
                      tb.grid_m, tb.norm, tb.max_radius, float(d.divergence_factor), int(d.divergence_run),
                      float(d.mu), B, 64, 1e-5, lab.data_ptr(), soft.data_ptr(), Tout.ctypes.data,
                      ws.data_ptr(), wsb, st.ctypes.data, s.cuda_stream)
            e1.record(s)
            torch.cuda.synchronize()
            host_ms.append(1e3 * (time.perf_counter() - h0))
            dev_ms.append(e0.elapsed_time(e1))
        it = int(st[0])
        print(f"nsym 2^{lg} B {B:4d}: dev {min(dev_ms[1:]):7.3f} ms host {min(host_ms[1:]):7.3f} ms "
              f"{nsym / min(dev_ms[1:]) / 1e6:7.3f} GBaud iters {it} fallback {st[2]} "
              f"per_iter {[(int(st[6 + 2 * i]), int(st[7 + 2 * i])) for i in range(min(it, 6))]}", flush=True)
