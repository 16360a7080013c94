"""Equaliser states the reference supports, at full length (2^30 samples of
the 10,000 km QPSK stream, device resident):
  clean   the widely-linear equaliser (the bench workload);
  linear  widely_linear=False (rx:71-78, rx:491-497 with g = 0): the same
          block-parallel solver with the linear affine maps;
  burst   a burst that trips the divergence guard (rx:484-490) mid-stream:
          the freeze is found inside the block-parallel solve (exact freeze
          point from per-block exceedance runs, then a parallel frozen-tap map).

    python tools/ddlms_modes_bench.py [--steps 3]
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
    import dataclasses

    for name in ("clean", "linear", "burst"):
        cfg_n = cfg
        if name == "linear":
            cfg_n = dataclasses.replace(cfg, ddlms=dataclasses.replace(cfg.ddlms, widely_linear=False))
        if name == "burst":
            x[n // 2: n // 2 + 600] *= 100.0
        times = []
        for i in range(args.steps + 1):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            pipe = rxdsp.RxPipeline(cfg_n, reference_symbols=pts)
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
        gbaud = int(lab.shape[0]) / (min(times) * 1e-3) / 1e9
        print(f"{name}: step {min(times):.2f} ms ({gbaud:.2f} GBaud), ddlms stage {stage['ddlms'] * 1e3:.2f} ms, frames {res[name][2]}, "
              f"diverged {pipe.diverged}", flush=True)


if __name__ == "__main__":
    main()
