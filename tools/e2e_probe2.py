"""Timeline of harness.receive_host_stream (async DDLMS) for one 2^N step."""
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import torch  # noqa: E402

from paper_2108_07001_b200.captures import load_capture, tile  # noqa: E402
from paper_2108_07001_b200.harness import receive_host_stream  # noqa: E402

log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
chunk = 1 << int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 25
frame = 1 << int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 28
cap = load_capture("c5_qpsk_10000km_tile")
codes, _ = tile(cap, 1 << log2n)
cfg = cap.pipeline_config(ddlms_frame_symbols=frame)
if len(sys.argv) > 4:
    import dataclasses
    cfg = dataclasses.replace(cfg, gpu=dataclasses.replace(cfg.gpu, ddlms_tail_min_symbols=1 << int(sys.argv[4])))
ref = cap.symbols()[:10000]
dev = torch.device("cuda", 0)
host = torch.from_numpy(codes).pin_memory()
staging = torch.empty(host.shape[0], dtype=torch.int16, device=dev)

# host-side time per pipeline phase (monkeypatched timers)
from paper_2108_07001_b200 import rxdsp  # noqa: E402
HT = {}


def _wrap(name):
    f = getattr(rxdsp.RxPipeline, name)

    def g(self, *a, **k):
        t = time.perf_counter()
        try:
            return f(self, *a, **k)
        finally:
            HT.setdefault(name, []).append(time.perf_counter() - t)
    setattr(rxdsp.RxPipeline, name, g)


from paper_2108_07001_b200 import harness  # noqa: E402


def _wrap_mod(mod, name):
    f = getattr(mod, name)

    def g(*a, **k):
        t = time.perf_counter()
        try:
            return f(*a, **k)
        finally:
            HT.setdefault(name, []).append(time.perf_counter() - t)
    setattr(mod, name, g)


_wrap_mod(harness, "_stream_receiver")
if os.environ.get("KK_PROBE_NO_D2H") == "1":      # collect frames without packing / shipping bits
    def _collect_only(st, bits_host, d2h, dev, max_frames=None, final=False):
        st["pipe"].drain_device(wait_stream=d2h, want_soft=False, max_frames=max_frames)
    harness._drain_bits = _collect_only
_MODE = os.environ.get("KK_PROBE_D2H_MODE")
if _MODE:
    def _partial(st, bits_host, d2h, dev, max_frames=None, final=False):
        lab, soft, _ = st["pipe"].drain_device(wait_stream=d2h, want_soft=False, max_frames=max_frames)
        if not lab.numel():
            return
        nb = (lab.numel() * 2 + 7) // 8
        with torch.cuda.stream(d2h):
            packed = torch.empty(nb, dtype=torch.uint8, device=dev)
            if _MODE in ("pack", "both"):
                _lib.call("kk_pack_bits", lab.data_ptr(), lab.numel(), 0, None, 0, 2,
                          st["tb"].point_label.ctypes.data, st["order"], packed.data_ptr(), d2h.cuda_stream)
            if _MODE in ("copy", "both"):
                bits_host[:nb].copy_(packed, non_blocking=True)
        lab.record_stream(d2h)
    harness._drain_bits = _partial
from paper_2108_07001_b200 import _lib  # noqa: E402
_orig_call = _lib.call


SOLVES = []


def _timed_call(name, *a):
    t = time.perf_counter()
    if name == "kk_ddlms_solve":
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record(torch.cuda.current_stream())
        try:
            return _orig_call(name, *a)
        finally:
            eb.record(torch.cuda.current_stream())
            SOLVES.append((t, time.perf_counter(), ea, eb, a[1]))
    try:
        return _orig_call(name, *a)
    finally:
        dt = time.perf_counter() - t
        if dt > 5e-4:
            HT.setdefault("lib:" + name, []).append(dt)


_lib.call = _timed_call
_orig_sync = rxdsp._sync_device


def _sync_dbg(head, ref, skip, dev):
    t = time.perf_counter()
    e = torch.cuda.Event()
    e.record(torch.cuda.current_stream(dev))
    e.synchronize()
    HT.setdefault("sync:stream_before", []).append(time.perf_counter() - t)
    return _orig_sync(head, ref, skip, dev)


rxdsp._sync_device = _sync_dbg
for _n in ("__init__", "expect", "_do_sync", "_run_kk", "_run_carrier", "_run_static", "_run_ddlms", "drain_device", "_submit_frame", "_wait_frames"):
    _wrap(_n)
for rep in range(4):
    HT.clear()
    tr = []
    ms0 = torch.cuda.memory_stats()
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record()
    h0 = time.perf_counter()
    pipe, bits, n = receive_host_stream(cfg, host, cap.half_lsb, ref, chunk_samples=chunk, staging=staging, trace=tr)
    evs = list(pipe._events)
    t1 = torch.cuda.Event(enable_timing=True)
    t1.record()
    torch.cuda.synchronize()
    tot = t0.elapsed_time(t1)
    ms1 = torch.cuda.memory_stats()
    print(f"rep {rep}: {tot:.2f} ms {n / tot / 1e6:.3f} GBaud host {1e3 * (time.perf_counter() - h0):.2f} ms",
          "device allocs", ms1.get("num_device_alloc", 0) - ms0.get("num_device_alloc", 0),
          "frees", ms1.get("num_device_free", 0) - ms0.get("num_device_free", 0),
          "retries", ms1.get("num_alloc_retries", 0) - ms0.get("num_alloc_retries", 0))
    if rep in (1, 3):
        for item in tr:
            if item[0] == "mark":
                print(f"  mark {item[1]} @ {t0.elapsed_time(item[3]):8.2f} host @ {1e3 * (item[2] - h0):8.2f}")
                continue
            if item[0] == "copy_start":
                print(f"  copies start @ {t0.elapsed_time(item[2]):8.2f} host @ {1e3 * (item[1] - h0):8.2f}")
                continue
            if item[0] == "d2h":
                print(f"  d2h done @ {t0.elapsed_time(item[2]):8.2f} host @ {1e3 * (item[1] - h0):8.2f}")
                continue
            i, ht, rd, fe, nj = item
            print(f"  chunk {i:3d}: copied @ {t0.elapsed_time(rd):8.2f} fed @ {t0.elapsed_time(fe):8.2f} "
                  f"host @ {1e3 * (ht - h0):8.2f} pending {nj}")
        print("  stats", [(s["k0"], s["nsym"], s.get("iterations")) for s in pipe.ddlms_stats])
        for (ht0, ht1, ea, eb, ns) in SOLVES[-4:]:
            print(f"  solve nsym {ns}: gpu {t0.elapsed_time(ea):8.2f} - {t0.elapsed_time(eb):8.2f}  "
                  f"host {1e3 * (ht0 - h0):8.2f} - {1e3 * (ht1 - h0):8.2f}")
        for name, e0, e1 in evs[:8]:
            print(f"  first events: {name} start {t0.elapsed_time(e0):8.2f} end {t0.elapsed_time(e1):8.2f}")
        for name, e0, e1 in pipe._events:
            if name == "ddlms" and e1.query():
                try:
                    print(f"  frame: start {t0.elapsed_time(e0):8.2f} end {t0.elapsed_time(e1):8.2f}")
                except Exception:
                    pass
        pipe._events = evs
        print("  stages", pipe.stage_seconds)
        for k_, v_ in HT.items():
            print("  host", k_, "n", len(v_), "total ms %.2f" % (1e3 * sum(v_)), "max ms %.2f" % (1e3 * max(v_)),
                  "top", ["%.2f" % (1e3 * x) for x in sorted(v_)[-4:]])
    pipe.release_buffers()
