"""One kk_bit_xcorr call (2^24-bit streams, FFT 2^25) for an ncu capture of the
frame-sync kernels (fft_pass_kernel, pack/product/peak/side)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2108_07001_b200.harness import frame_sync_device  # noqa: E402

dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(1)
tx = torch.randint(0, 2, (1 << 24,), dtype=torch.uint8, device=dev, generator=g)
rx = tx[12345:12345 + (1 << 23)].clone()
for _ in range(2):
    lag, _, _ = frame_sync_device(rx, tx)
torch.cuda.synchronize()
print("lag", lag)
