"""Times K1 (kk_reconstruct_pairs) alone over a device-resident 2^30-sample
int16 stream (CUDA events, best of N) -- for comparing build variants
(KKB200_LIB=<variant .so>)."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    import numpy as np
    import torch

    from paper_2108_07001_b200 import _lib
    from paper_2108_07001_b200.captures import load_capture, tile

    cap = load_capture("c5_qpsk_10000km_tile")
    n = 1 << 30
    codes, _ = tile(cap, n)
    x = torch.from_numpy(codes).cuda()
    hop = 512
    nh = n // hop
    out = torch.empty(n, dtype=torch.complex64, device="cuda")
    hs = torch.empty(nh, dtype=torch.complex64, device="cuda")
    hd = torch.empty(nh, dtype=torch.uint8, device="cuda")
    su = torch.zeros(hop, device="cuda"); sa = torch.zeros(hop // 2, device="cuda")
    sd = torch.zeros(hop // 2, dtype=torch.uint8, device="cuda")
    nu = torch.empty(hop, device="cuda"); na = torch.empty(hop // 2, device="cuda")
    nd = torch.empty(hop // 2, dtype=torch.uint8, device="cuda")
    cl = torch.zeros(1, dtype=torch.int64, device="cuda")
    tab = torch.from_numpy(np.exp(-2j * np.pi * np.arange(1000) / 1000).astype(np.complex64)).cuda()
    s = torch.cuda.current_stream().cuda_stream
    p = lambda t: t.data_ptr()
    ts = []
    for i in range(8):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.call("kk_reconstruct_pairs", 0, p(x), cap.half_lsb, 1e-12, nh, p(su), p(sa), p(sd), p(nu), p(na), p(nd),
                  p(out), p(hs), p(hd), p(cl), 0, 129, 1000, p(tab), 0, 1, s)
        e1.record()
        torch.cuda.synchronize()
        if i:
            ts.append(e0.elapsed_time(e1))
    ck = float(torch.view_as_real(out[:1 << 20]).double().abs().sum())
    print(f"{os.environ.get('KKB200_LIB', 'main')}: K1 {min(ts):.3f} ms (median {sorted(ts)[len(ts)//2]:.3f}) "
          f"checksum {ck:.6e}", flush=True)


if __name__ == "__main__":
    main()
