"""Timeline probe of the end-to-end host-stream receive (bench e2e leg):
raw pinned H2D bandwidth, then one receive_host_stream step with the copy
events and per-feed compute markers printed relative to the step start."""
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import torch  # noqa: E402

from paper_2108_07001_b200 import _lib, harness, rxdsp  # noqa: E402
from paper_2108_07001_b200.constellation import slicer_tables  # noqa: E402
from paper_2108_07001_b200.captures import load_capture, tile  # noqa: E402
from paper_2108_07001_b200.sigcore import AdcCodes  # noqa: E402

log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
chunk = 1 << int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 25
frame = 1 << int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 28
cap = load_capture("c5_qpsk_10000km_tile")
codes, _ = tile(cap, 1 << log2n)
cfg = cap.pipeline_config(ddlms_frame_symbols=frame)
ref = cap.symbols()[:10000]
dev = torch.device("cuda", 0)
tb = slicer_tables(4)
host = torch.from_numpy(codes).pin_memory()
dst = torch.empty(host.shape[0], dtype=torch.int16, device=dev)
for _ in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    dst.copy_(host, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"H2D {host.numel() * 2 / 1e9:.2f} GB in {ms:.2f} ms = {host.numel() * 2 / ms / 1e6:.1f} GB/s")
lab_host = torch.empty(host.shape[0] // 4 + 8, dtype=torch.uint8).pin_memory()
t = torch.empty(host.shape[0] // 4 + 8, dtype=torch.uint8, device=dev)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
lab_host.copy_(t, non_blocking=True)
e1.record()
torch.cuda.synchronize()
print(f"D2H {t.numel() / 1e9:.3f} GB in {e0.elapsed_time(e1):.2f} ms")

# instrumented copy of harness.receive_host_stream
for rep in range(3):
    comp = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(device=dev)
    d2h = torch.cuda.Stream(device=dev)
    n = host.shape[0]
    starts = list(range(0, n, chunk))
    ready = [torch.cuda.Event(enable_timing=True) for _ in starts]
    fed = [torch.cuda.Event(enable_timing=True) for _ in starts]
    t_start = torch.cuda.Event(enable_timing=True)
    t_start.record(comp)
    h0 = time.perf_counter()
    pipe = rxdsp.RxPipeline(cfg, reference_symbols=ref, device=dev)
    pipe.expect(host.shape[0], chunk)
    copy.wait_stream(comp)
    with torch.cuda.stream(copy):
        for i, a in enumerate(starts):
            m = min(chunk, n - a)
            dst[a:a + m].copy_(host[a:a + m], non_blocking=True)
            ready[i].record(copy)
    n_out = 0
    b_out = 0
    host_t = []
    d2h_ev = []
    for i, a in enumerate(starts):
        m = min(chunk, n - a)
        comp.wait_event(ready[i])
        pipe.feed(AdcCodes(dst[a:a + m], cap.half_lsb, cfg.adc_rate_hz), flush=i == len(starts) - 1)
        fed[i].record(comp)
        host_t.append(time.perf_counter() - h0)
        lab, _, _ = pipe.drain_device()
        if lab.numel():
            nb = (lab.numel() * 2 + 7) // 8
            packed = torch.empty(nb, dtype=torch.uint8, device=dev)
            _lib.call("kk_pack_bits", lab.data_ptr(), lab.numel(), n_out, None, 0, 2,
                      tb.point_label.ctypes.data, 4, packed.data_ptr(), comp.cuda_stream)
            d2h.wait_stream(comp)
            with torch.cuda.stream(d2h):
                lab_host[b_out:b_out + nb].copy_(packed, non_blocking=True)
                ev = torch.cuda.Event(enable_timing=True)
                ev.record(d2h)
                d2h_ev.append((i, lab.numel(), ev))
            packed.record_stream(d2h)
            n_out += lab.numel()
            b_out += nb
    comp.wait_stream(d2h)
    t_end = torch.cuda.Event(enable_timing=True)
    t_end.record(comp)
    torch.cuda.synchronize()
    tot = t_start.elapsed_time(t_end)
    print(f"rep {rep}: total {tot:.2f} ms, symbols {n_out}, {n_out / tot / 1e6:.3f} GBaud")
    if rep == 2:
        for i in range(len(starts)):
            print(f"  chunk {i:3d}: copied @ {t_start.elapsed_time(ready[i]):8.2f}  fed @ "
                  f"{t_start.elapsed_time(fed[i]):8.2f}  host @ {host_t[i] * 1e3:8.2f}")
        for i, nn, ev in d2h_ev:
            print(f"  d2h after chunk {i}: {nn} labels done @ {t_start.elapsed_time(ev):8.2f}")
        print("  stages", pipe.stage_seconds)
    pipe.release_buffers()
