"""Kernel timeline of one bench step (the device-resident 2^30-sample receive)
from the CUDA profiler activity trace (torch.profiler / CUPTI; nsys is not
installed in this image).  Prints every kernel / memcpy with its start,
duration and the idle gap before it, and a summary: device busy time, idle
time, and the largest gaps -- the host-side overhead the step pays outside
the kernels.

    python tools/step_timeline.py [--format c5_qpsk_10000km_tile] [--out gpurun_out/timeline.txt]
"""

from __future__ import annotations

import argparse
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--format", default="c5_qpsk_10000km_tile")
    ap.add_argument("--samples-log2", type=int, default=30)
    ap.add_argument("--out", default=None)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()

    import torch
    from torch.profiler import ProfilerActivity, profile

    from paper_2108_07001_b200 import superframe
    from paper_2108_07001_b200.captures import load_capture, tile
    from paper_2108_07001_b200.harness import device_ber
    from paper_2108_07001_b200.sigcore import AdcCodes

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    cap = load_capture(args.format)
    cfg = cap.pipeline_config()
    n = 1 << args.samples_log2
    job = superframe.plan_superframe(0, 1, n)
    codes, _ = tile(cap, n)
    codes_dev = torch.from_numpy(codes).to(dev)
    ref_dev = torch.from_numpy(tile(cap, n)[1]).to(dev)
    pts = cap.symbols()[:max(cfg.sync_symbols, cfg.ddlms.startup_symbols)]

    def step():
        r = superframe.receive_superframe(cfg, AdcCodes(codes_dev, cap.half_lsb), pts, job)
        lab = r.labels
        e, c = device_ber(lab, ref_dev[:lab.shape[0]], cap.order, cfg.ddlms.startup_symbols + 2048,
                          lab.shape[0] - 4096, tile_symbols=len(cap.sym_idx), seam_guard=128)
        return r

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        torch.cuda.synchronize()
        for _ in range(2):             # two back-to-back steps: the gap between them counts too
            step()
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ev.sort(key=lambda e: e.time_range.start)
    lines = []
    t_first = ev[0].time_range.start
    busy = 0.0
    gaps = []
    prev_end = t_first
    for e in ev:
        s, d = e.time_range.start, e.time_range.elapsed_us()
        gap = s - prev_end
        if gap > 0:
            gaps.append((gap, e.name[:60], s - t_first))
        busy += d
        lines.append(f"{(s - t_first) / 1e3:9.3f} ms  {d:9.1f} us  gap {max(gap, 0):8.1f} us  {e.name[:90]}")
        prev_end = max(prev_end, s + d)
    span = prev_end - t_first
    gaps.sort(reverse=True)
    summ = [f"2 steps; kernels/copies: {len(ev)}", f"span (first start -> last end): {span / 1e3:.3f} ms",
            f"device busy: {busy / 1e3:.3f} ms   idle: {(span - busy) / 1e3:.3f} ms",
            "largest idle gaps (us, before kernel, at ms):"]
    summ += [f"  {g:9.1f}  {nm}  @{at / 1e3:.3f}" for g, nm, at in gaps[:15]]
    text = "\n".join(summ + ["", *lines])
    print("\n".join(summ))
    if args.out:
        os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
        with open(args.out, "w") as f:
            f.write(text + "\n")


if __name__ == "__main__":
    main()
