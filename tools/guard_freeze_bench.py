"""Device-resident receive of the 2^30-sample 10,000 km QPSK stream with a
burst that trips the divergence guard (rx:484-490) mid-stream, vs the same
stream without it: the freeze is handled inside the block-parallel solve
(exact freeze point from the per-block exceedance runs, then a parallel
frozen-tap map), so the frame costs about the same as a normal one.

    python tools/guard_freeze_bench.py [--steps 3]
"""
import argparse
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    import torch

    from paper_2108_07001_b200 import rxdsp
    from paper_2108_07001_b200.captures import load_capture, tile

    cap = load_capture("c5_qpsk_10000km_tile")
    cfg = cap.pipeline_config()
    n = 1 << 30
    codes, _ = tile(cap, n)
    x = torch.from_numpy(codes).cuda().float() * cap.half_lsb          # f32 input (the burst exceeds 12 bits)
    pts = cap.symbols()[:10000]
    res = {}
    for name in ("clean", "burst"):
        if name == "burst":
            x[n // 2: n // 2 + 600] *= 100.0
        times = []
        for i in range(args.steps + 1):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            pipe = rxdsp.RxPipeline(cfg, reference_symbols=pts)
            pipe.feed(x, flush=True)
            lab, _, _ = pipe.drain_device()
            e1.record()
            torch.cuda.synchronize()
            if i:
                times.append(e0.elapsed_time(e1))
            st = pipe.ddlms_stats
            stage = pipe.stage_seconds
            pipe.release_buffers()
        res[name] = (min(times), stage["ddlms"] * 1e3, [(s["mode"], s.get("iterations")) for s in st],
                     pipe.diverged)
        print(f"{name}: step {min(times):.2f} ms, ddlms stage {stage['ddlms'] * 1e3:.2f} ms, frames {res[name][2]}, "
              f"diverged {pipe.diverged}", flush=True)


if __name__ == "__main__":
    main()
