"""Which small transfers on a second stream wait for bulk host->device copies
queued on another stream?  (Shapes the ingest ordering of
harness.receive_host_stream.)  Prints host ms until each probe completes."""
import time

import numpy as np
import torch

dev = torch.device("cuda", 0)
n = 1 << 30
host = torch.empty(n, dtype=torch.int16).pin_memory()
dst = torch.empty(n, dtype=torch.int16, device=dev)
small_np = np.arange(4096, dtype=np.float32)
small_pin = torch.from_numpy(small_np).pin_memory()
small_dev = torch.empty(4096, dtype=torch.float32, device=dev)
rb_pin = torch.empty(16, dtype=torch.float32).pin_memory()
bulk = torch.cuda.Stream(device=dev)
other = torch.cuda.Stream(device=dev)
chunk = 1 << 25


def run(name, probe):
    torch.cuda.synchronize()
    with torch.cuda.stream(bulk):
        for a in range(0, n, chunk):
            dst[a:a + chunk].copy_(host[a:a + chunk], non_blocking=True)
    t0 = time.perf_counter()
    with torch.cuda.stream(other):
        probe()
    t1 = time.perf_counter()
    ev = torch.cuda.Event()
    ev.record(other)
    ev.synchronize()
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"{name:40s} host call {1e3 * (t1 - t0):7.2f} ms  done {1e3 * (t2 - t0):7.2f} ms  bulk done {1e3 * (t3 - t0):7.2f} ms",
          flush=True)


for rep in range(2):
    run("kernel only", lambda: small_dev.mul_(2))
    run("H2D pinned non_blocking", lambda: small_dev.copy_(small_pin, non_blocking=True))
    run("H2D pageable", lambda: small_dev.copy_(torch.from_numpy(small_np)))
    run("H2D pin_memory().to(non_blocking)", lambda: torch.from_numpy(small_np).pin_memory().to(dev, non_blocking=True))
    run("D2H small to pinned", lambda: rb_pin.copy_(small_dev[:16], non_blocking=True))
    run("D2H small pageable", lambda: small_dev[:16].cpu())
    run("kernel + D2H pinned", lambda: (small_dev.mul_(2), rb_pin.copy_(small_dev[:16], non_blocking=True)))


def staged(name, upload_bytes, pinned, wait_upload=True, wait_chunk0=False, timing=False):
    """2 bulk chunks, then an upload on `other`, then the rest of the bulk
    copies, then a kernel + small D2H readback on `other`."""
    torch.cuda.synchronize()
    a_np = np.ones(upload_bytes // 4, np.float32)
    t0 = time.perf_counter()
    ev0 = torch.cuda.Event(enable_timing=timing)
    with torch.cuda.stream(bulk):
        for a in range(0, 2 * chunk, chunk):
            dst[a:a + chunk].copy_(host[a:a + chunk], non_blocking=True)
            if a == 0:
                ev0.record(bulk)
    with torch.cuda.stream(other):
        if pinned:
            u = torch.from_numpy(a_np).pin_memory().to(dev, non_blocking=True)
        else:
            u = torch.from_numpy(a_np).to(dev)
        ev = torch.cuda.Event()
        ev.record(other)
    t1 = time.perf_counter()
    if wait_upload:
        ev.synchronize()
    t2 = time.perf_counter()
    with torch.cuda.stream(bulk):
        for a in range(2 * chunk, n, chunk):
            dst[a:a + chunk].copy_(host[a:a + chunk], non_blocking=True)
    t3 = time.perf_counter()
    with torch.cuda.stream(other):
        if wait_chunk0:
            other.wait_event(ev0)
        u.mul_(2)
        rb_pin.copy_(u[:16], non_blocking=True)
        ev2 = torch.cuda.Event()
        ev2.record(other)
    ev2.synchronize()
    t4 = time.perf_counter()
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    print(f"{name:44s} upload call {1e3 * (t1 - t0):6.2f} waited {1e3 * (t2 - t0):6.2f} queued {1e3 * (t3 - t0):6.2f} "
          f"readback {1e3 * (t4 - t0):6.2f} bulk {1e3 * (t5 - t0):6.2f} ms", flush=True)


for rep in range(2):
    for ub in (16 << 10, 64 << 10, 128 << 10, 1 << 20):
        staged(f"pinned upload {ub >> 10} KB", ub, True)
        staged(f"pageable upload {ub >> 10} KB", ub, False)
    staged("pinned 128 KB, no wait", 128 << 10, True, False)
    staged("pinned 128 KB, wait chunk0 event", 128 << 10, True, True, True)
    staged("pinned 128 KB, wait chunk0 timing event", 128 << 10, True, True, True, True)
    staged("pageable 16 KB, wait chunk0 timing event", 16 << 10, False, True, True, True)
