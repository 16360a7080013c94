"""Host-side profile of one end-to-end streaming receive step
(harness.receive_host_stream, packed 12-bit, 2^30 samples): wall time of the
call, time until the first K1 launch is enqueued, and the top cumulative
Python functions (cProfile) -- the host work on the e2e critical path.

    python tools/e2e_host_profile.py
"""
import cProfile
import dataclasses
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2108_07001_b200 import _lib  # noqa: E402
from paper_2108_07001_b200.captures import load_capture, tile  # noqa: E402
from paper_2108_07001_b200.harness import receive_host_stream  # noqa: E402
from paper_2108_07001_b200.sigcore import pack12  # noqa: E402

cap = load_capture("c5_qpsk_10000km_tile")
cfg = cap.pipeline_config()
cfg = dataclasses.replace(cfg, gpu=dataclasses.replace(cfg.gpu, ddlms_frame_symbols=1 << 26))
codes, _ = tile(cap, 1 << 30)
host = torch.from_numpy(pack12(codes)).pin_memory()
pts = cap.symbols()[:10000]
bits = torch.empty((1 << 30) // 4 * 2 // 8 + 65536, dtype=torch.uint8).pin_memory()
st = torch.empty(3 << 29, dtype=torch.uint8, device="cuda")

# first K1 enqueue time: wrap the library entry points
lib = _lib.load()
marks = {}
t_call = [0.0]
spent = {}
lastm = {}


def wrap(name):
    f = getattr(lib, name)

    def g(*a):
        t0 = time.perf_counter()
        marks.setdefault(name, t0 - t_call[0])
        r = f(*a)
        c, tt, mx = spent.get(name, (0, 0.0, 0.0))
        d = time.perf_counter() - t0
        spent[name] = (c + 1, tt + d, max(mx, d))
        lastm[name] = t0 - t_call[0]
        return r
    g.argtypes, g.restype = f.argtypes, f.restype
    setattr(lib, name, g)


for nm in ("kk_reconstruct_pairs", "kk_static_blocks", "kk_ddlms_solve_async", "kk_pack_bits", "kk_upload"):
    wrap(nm)


def step():
    return receive_host_stream(cfg, host, cap.half_lsb, pts, chunk_samples=1 << 25, bits_host=bits, staging=st,
                               packed12_samples=1 << 30)


for i in range(4):
    marks.clear()
    spent.clear()
    torch.cuda.synchronize()
    t_call[0] = time.perf_counter()
    pipe, bh, n = step()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t_call[0]
    print(f"step {i}: {dt * 1e3:.1f} ms; first enqueue (ms after call): "
          + ", ".join(f"{k} {v * 1e3:.2f}" for k, v in sorted(marks.items(), key=lambda kv: kv[1])), flush=True)
    print("   last enqueue (ms):", {k: round(v * 1e3, 2) for k, v in lastm.items()})
    print("   host time in library calls:", {k: (c, round(tt * 1e3, 2), round(mx * 1e3, 2)) for k, (c, tt, mx) in
                                         spent.items()}, flush=True)
    pipe.release_buffers()

pr = cProfile.Profile()
torch.cuda.synchronize()
pr.enable()
pipe, bh, n = step()
torch.cuda.synchronize()
pr.disable()
pipe.release_buffers()
pstats.Stats(pr).sort_stats("cumulative").print_stats(35)
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
