"""Wall-clock breakdown of one bench step (syncs between phases) to locate
host-side overhead next to the device stage times."""
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
codes, _ = tile(cap, 1 << log2n)
cfg = cap.pipeline_config()
ref = cap.symbols()[:10000]
cd = torch.from_numpy(codes).cuda()
for rep in range(3):
    torch.cuda.synchronize()
    T = {}
    t = time.perf_counter()
    pipe = rxdsp.RxPipeline(cfg, reference_symbols=ref)
    torch.cuda.synchronize(); T["init"] = time.perf_counter() - t; t = time.perf_counter()
    x, dt, sc = rxdsp._as_device_input(AdcCodes(cd, cap.half_lsb), pipe.dev)
    pipe._append_raw(x, dt, sc)
    n_hops = x.shape[0] // 512
    pipe._run_kk(pipe._raw[:n_hops * 512], n_hops)
    pipe._raw = pipe._raw[n_hops * 512:]
    torch.cuda.synchronize(); T["kk"] = time.perf_counter() - t; t = time.perf_counter()
    pipe._run_carrier(True)
    torch.cuda.synchronize(); T["carrier"] = time.perf_counter() - t; t = time.perf_counter()
    pipe._run_static(True)
    torch.cuda.synchronize(); T["static"] = time.perf_counter() - t; t = time.perf_counter()
    pipe._do_sync(True)
    torch.cuda.synchronize(); T["sync"] = time.perf_counter() - t; t = time.perf_counter()
    pipe._run_ddlms(True)
    torch.cuda.synchronize(); T["ddlms"] = time.perf_counter() - t; t = time.perf_counter()
    lab, soft, meta = pipe.drain_device()
    pipe.release_buffers()
    torch.cuda.synchronize(); T["drain"] = time.perf_counter() - t
    print(rep, {k: round(v * 1e3, 2) for k, v in T.items()}, "total", round(sum(T.values()) * 1e3, 2),
          pipe.ddlms_stats[-1].get("per_iter"))
