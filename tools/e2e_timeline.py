"""Kernel/copy timeline of one end-to-end host-stream receive
(harness.receive_host_stream) from the CUPTI activity trace (torch.profiler;
nsys is absent): per stream, the first start / last end and busy time, and
the launches in time order with their stream.

    python tools/e2e_timeline.py [--out gpurun_out/e2e_timeline.txt]
"""

from __future__ import annotations

import argparse
import dataclasses
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--format", default="c5_qpsk_10000km_tile")
    ap.add_argument("--packed12", action="store_true")
    args = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile

    from paper_2108_07001_b200.captures import load_capture, tile
    from paper_2108_07001_b200.harness import receive_host_stream

    cap = load_capture(args.format)
    cfg = cap.pipeline_config()
    cfg = dataclasses.replace(cfg, gpu=dataclasses.replace(cfg.gpu, ddlms_frame_symbols=1 << 25))   # as bench.py e2e
    n = 1 << 30
    codes, _ = tile(cap, n)
    from paper_2108_07001_b200.sigcore import pack12

    host = torch.from_numpy(pack12(codes) if args.packed12 else codes).pin_memory()
    pts = cap.symbols()[:10000]
    bits = torch.empty(n // 4 * 2 // 8 + 65536, dtype=torch.uint8).pin_memory()
    st = (torch.empty(3 * n // 2, dtype=torch.uint8, device="cuda") if args.packed12
          else torch.empty(n, dtype=torch.int16, device="cuda"))

    def step():
        pipe, _, _ = receive_host_stream(cfg, host, cap.half_lsb, pts, chunk_samples=1 << 25, bits_host=bits,
                                         staging=st, packed12_samples=n if args.packed12 else None)
        pipe.release_buffers()

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        step()
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ev.sort(key=lambda e: e.time_range.start)
    t0 = ev[0].time_range.start
    per = {}
    lines = []
    for e in ev:
        sid = getattr(e, "device_resource_id", -1)
        s, d = e.time_range.start - t0, e.time_range.elapsed_us()
        a = per.setdefault(sid, [s, s + d, 0.0, 0])
        a[0] = min(a[0], s)
        a[1] = max(a[1], s + d)
        a[2] += d
        a[3] += 1
        lines.append(f"{s / 1e3:9.3f} ms {d:9.1f} us  stream {sid:4d}  {e.name[:80]}")
    summ = [f"span {max(a[1] for a in per.values()) / 1e3:.3f} ms"]
    for sid, a in sorted(per.items()):
        summ.append(f"stream {sid}: {a[3]} ops, {a[0] / 1e3:.3f} .. {a[1] / 1e3:.3f} ms, busy {a[2] / 1e3:.3f} ms")
    print("\n".join(summ))
    if args.out:
        with open(args.out, "w") as f:
            f.write("\n".join(summ + [""] + lines) + "\n")


if __name__ == "__main__":
    main()
