"""Device-resident receive throughput and BER per modulation format
(BASELINE configs[1], [2], [4]): a 2^N-sample continuous capture of each
golden configuration's link generated on the GPU (capgen), received in one
feed, timed with CUDA events (median of 3 after a warm-up)."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2108_07001_b200 import capgen, rxdsp  # noqa: E402
from paper_2108_07001_b200.captures import load_capture  # noqa: E402
from paper_2108_07001_b200.constellation import make_constellation  # noqa: E402
from paper_2108_07001_b200.harness import device_ber  # noqa: E402
from paper_2108_07001_b200.sigcore import AdcCodes  # noqa: E402

log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
names = sys.argv[2].split(",") if len(sys.argv) > 2 else ["c2_16qam_5600km_rel-20", "c3_64qam_1600km_rel-20",
                                                         "c5_qpsk_10000km_tile"]
dev = torch.device("cuda", 0)
for name in names:
    cap = load_capture(name)
    c = cap.meta["config"]
    gen = capgen.CaptureGenerator(capgen.GenParams.from_config(c), seed=7, device=dev)
    n_sym = (1 << log2n) // 4
    codes, half, idx, _ = gen.generate(n_sym, chunk_symbols=1 << 20)
    pts = make_constellation(cap.order).points
    gpu_kw = {}
    if os.environ.get("KK_DDLMS_BLOCK"):
        gpu_kw["ddlms_block"] = int(os.environ["KK_DDLMS_BLOCK"])
    if os.environ.get("KK_FRAME_LOG2"):
        gpu_kw["ddlms_frame_symbols"] = 1 << int(os.environ["KK_FRAME_LOG2"])
    cfg = cap.pipeline_config(**gpu_kw)
    ref = pts[idx[:max(cfg.sync_symbols, cfg.ddlms.startup_symbols)]]
    ref_dev = torch.from_numpy(idx.astype(np.uint8)).to(dev)
    times = []
    for rep in range(4):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pipe = rxdsp.RxPipeline(cfg, reference_symbols=ref, device=dev)
        pipe.feed(AdcCodes(codes, half, 4e9), flush=True)
        lab, _, meta = pipe.drain_device(want_soft=False)
        e1.record()
        torch.cuda.synchronize()
        if rep:
            times.append(e0.elapsed_time(e1))
        stats = pipe.ddlms_stats
        print("   rep", rep, "iterations", [s_.get("iterations") for s_ in stats], "fallback",
              [s_.get("fallback") for s_ in stats], "labels hash", int(lab.to(torch.int64).sum().item()), flush=True)
        pipe.release_buffers()
    k0 = meta[0][0]
    head = cfg.ddlms.startup_symbols + 2048
    errs, cnt = device_ber(lab, ref_dev[k0:k0 + lab.shape[0]], cap.order, head, lab.shape[0] - 4096)
    k = make_constellation(cap.order).bits_per_symbol
    ms = float(np.median(times))
    print(f"{name}: {lab.numel() / ms / 1e6:.3f} GBaud ({ms:.2f} ms for 2^{log2n} samples), "
          f"BER {int(errs.item()) / (int(cnt.item()) * k):.3e} over {int(cnt.item()) * k} bits "
          f"(reference point {cap.meta['point']['ber']:.3e}), DDLMS iterations {[s.get('iterations') for s in stats]} "
          f"fallback {[s.get('fallback') for s in stats]} per_iter {[s.get('per_iter') for s in stats]}",
          flush=True)
    del codes
