"""Time kk_bit_xcorr (frame_sync's all-lag bit correlation)
on the GPU against the reference formula on the host (numpy/scipy float64
FFT, metrics.py frame_sync :69-112) for a few stream lengths.

    python tools/xcorr_bench.py
"""

import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2108_07001_b200 import _lib  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    st = torch.cuda.current_stream()
    g = torch.Generator(device=dev).manual_seed(1)
    for log_bits in (20, 24, 26, 28, 29):
        n_tx = 1 << log_bits
        lag = n_tx // 7
        n_rx = n_tx - lag - 64
        tx = torch.randint(0, 2, (n_tx,), dtype=torch.uint8, device=dev, generator=g)
        rx = tx[lag:lag + n_rx].clone()
        nws = int(_lib.load().kk_bit_xcorr_workspace_bytes(n_rx, n_tx, 0))
        ws = torch.empty(nws, dtype=torch.uint8, device=dev)
        out = torch.empty(3, dtype=torch.int64, device=dev)

        def run():
            _lib.call("kk_bit_xcorr", rx.data_ptr(), n_rx, tx.data_ptr(), n_tx, 0, ws.data_ptr(), nws,
                      out.data_ptr(), st.cuda_stream)

        for _ in range(2):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        e0.record()
        for _ in range(reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        k, peak, side = (int(v) for v in out.cpu())
        nfft = 1
        while nfft < n_rx + n_tx - 1:
            nfft <<= 1
        log_n = nfft.bit_length() - 1
        passes = 2 * ((log_n + 9) // 10)
        gbs = passes * 32 * nfft / (ms * 1e-3) / 1e9
        ok = (n_tx - 1 - k == lag) and peak == n_rx
        line = (f"bits 2^{log_bits}: FFT 2^{log_n}, {passes} Stockham passes, {ms:8.2f} ms "
                f"({gbs:6.0f} GB/s pass traffic), lag ok {ok}, ratio {peak / max(side, 1):.0f}")
        if log_bits <= 24:
            from scipy.signal import fftconvolve
            a = rx.cpu().numpy().astype(np.float64) * 2 - 1
            b = tx.cpu().numpy().astype(np.float64) * 2 - 1
            t0 = time.perf_counter()
            fftconvolve(a, b[::-1], mode="full")
            line += f"; host scipy fftconvolve {1e3 * (time.perf_counter() - t0):.0f} ms"
        print(line, flush=True)
        del ws


if __name__ == "__main__":
    main()
