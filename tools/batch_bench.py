"""Sweep-style batch receive: every golden capture (262,144
ADC samples each) received sequentially vs concurrently (receive_batch)."""
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2108_07001_b200 import rxdsp  # noqa: E402
from paper_2108_07001_b200.captures import list_captures, load_capture  # noqa: E402
from paper_2108_07001_b200.harness import receive_batch  # noqa: E402

names = [n for n in list_captures() if n.startswith(("c1", "c2", "c3", "c4")) and not n.endswith("_tile")]
caps = [load_capture(n) for n in names]
items = [(c.pipeline_config(), c.adc, c.symbols()) for c in caps]
nsyms = 0


def seq():
    n = 0
    for cfg, adc, ref in items:
        p = rxdsp.RxPipeline(cfg, reference_symbols=ref)
        p.feed(adc)
        p.feed(np.zeros(0), flush=True)
        lab, _, _ = p.drain_device()
        n += lab.numel()
    torch.cuda.synchronize()
    return n


def bat(conc):
    r = receive_batch(items, max_concurrency=conc)
    torch.cuda.synchronize()
    return sum(x[0].numel() for x in r)


for f, lab in ((seq, "sequential"), (lambda: bat(None), "batched")):
    f()
    t = time.perf_counter()
    reps = 3
    for _ in range(reps):
        n = f()
    dt = (time.perf_counter() - t) / reps
    print(f"{lab:12s}: {len(items)} streams, {n} symbols, {dt * 1e3:.1f} ms, {n / dt / 1e6:.2f} MBaud aggregate")
