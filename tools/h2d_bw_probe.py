"""Host->device bandwidth of a 2 GiB pinned int16 stream copied in chunks:
one copy stream vs several concurrent ones (does a second copy engine add
PCIe throughput?)."""
import torch

dev = torch.device("cuda", 0)
n = 1 << 30
host = torch.empty(n, dtype=torch.int16).pin_memory()
dst = torch.empty(n, dtype=torch.int16, device=dev)
streams = [torch.cuda.Stream(device=dev) for _ in range(4)]
for chunk_log2 in (23, 25):
    chunk = 1 << chunk_log2
    for ns in (1, 2, 4):
        best = 0.0
        for rep in range(4):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for s in streams[:ns]:
                s.wait_stream(torch.cuda.current_stream())
            for i, a in enumerate(range(0, n, chunk)):
                with torch.cuda.stream(streams[i % ns]):
                    dst[a:a + chunk].copy_(host[a:a + chunk], non_blocking=True)
            for s in streams[:ns]:
                torch.cuda.current_stream().wait_stream(s)
            e1.record()
            torch.cuda.synchronize()
            best = max(best, 2 * n / e0.elapsed_time(e1) / 1e6)
        print(f"chunk 2^{chunk_log2} streams {ns}: {best:6.2f} GB/s", flush=True)
