"""GPU measurement kernels against the reference's
formulas: frame_sync's all-lag bipolar cross-correlation (metrics.py
frame_sync :69-112) through kk_bit_xcorr, labels -> bits, per-window error
counts (metrics.py windowed_q :130-150) and the EVM sums (metrics.py evm
:169-179).

The correlation of two +-1 streams is an integer; the expected peak index,
peak and sidelobe magnitudes are computed here with scipy's float64
fftconvolve rounded to integers (what the reference evaluates, exact at these
sizes) and must agree exactly.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from scipy.signal import fftconvolve  # noqa: E402

from paper_2108_07001_b200 import _lib  # noqa: E402
from paper_2108_07001_b200.harness import frame_sync_device  # noqa: E402
from paper_2108_07001_b200.metrics import SyncFailure, frame_sync  # noqa: E402


def _expected(rx, tx, circular):
    a = rx.astype(np.float64) * 2 - 1
    b = tx.astype(np.float64) * 2 - 1
    if circular:
        c = np.rint(np.fft.ifft(np.fft.fft(a) * np.conj(np.fft.fft(b))).real).astype(np.int64)
        w = 0
    else:
        c = np.rint(fftconvolve(a, b[::-1], mode="full")).astype(np.int64)
        w = 2
    mag = np.abs(c)
    k = int(np.argmax(mag))
    side = np.delete(mag, np.arange(max(0, k - w), min(len(mag), k + w + 1)))
    return k, int(mag[k]), int(side.max())


def _xcorr(rx, tx, circular):
    dev = torch.device("cuda:0")
    r = torch.from_numpy(rx).to(dev)
    t = torch.from_numpy(tx).to(dev)
    nws = int(_lib.load().kk_bit_xcorr_workspace_bytes(len(rx), len(tx), int(circular)))
    ws = torch.empty(nws, dtype=torch.uint8, device=dev)
    out = torch.empty(3, dtype=torch.int64, device=dev)
    _lib.call("kk_bit_xcorr", r.data_ptr(), len(rx), t.data_ptr(), len(tx), int(circular), ws.data_ptr(), nws,
              out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    return tuple(int(v) for v in out.cpu())


def _streams(rng, n_rx, n_tx, lag, flip=0.05):
    """tx random; rx = tx[lag:] (or padded for negative lag) with bit flips."""
    tx = rng.integers(0, 2, n_tx, dtype=np.uint8)
    if lag >= 0:
        rx = tx[lag:lag + n_rx].copy()
    else:
        rx = np.concatenate([rng.integers(0, 2, -lag, dtype=np.uint8), tx[: n_rx + lag]])
    if len(rx) < n_rx:
        rx = np.concatenate([rx, rng.integers(0, 2, n_rx - len(rx), dtype=np.uint8)])
    rx ^= (rng.random(n_rx) < flip).astype(np.uint8)
    return rx, tx


# correlation lengths spanning FFT sizes 2^15 .. 2^23 (every pass split of
# the Stockham plan: 8+7, 8+8, 9+8, 9+9, 10+9, 10+10, 7+7+7, 8+7+7, 8+8+7)
@pytest.mark.parametrize("n_rx,n_tx,lag", [
    (9000, 1 << 14, 1234), (1 << 14, 1 << 14, -700), (40000, 50000, 9999), (70000, 1 << 16, -3),
    (150000, 1 << 17, 77777), (1 << 18, 300000, 5), (600000, 1 << 19, -12345), (1 << 20, 1 << 20, 0),
    (3_000_001, 2_500_000, 1_000_000)])
def test_bit_xcorr_exact_linear(n_rx, n_tx, lag):
    rng = np.random.default_rng(n_rx ^ n_tx)
    rx, tx = _streams(rng, n_rx, n_tx, lag)
    if n_rx == n_tx:   # keep the linear path: drop one bit
        rx = rx[:-1]
    assert _xcorr(rx, tx, False) == _expected(rx, tx, False)


@pytest.mark.parametrize("n,shift", [(1 << 14, 5), (20011, 19000), (1 << 17, 0), (777_777, 123_456)])
def test_bit_xcorr_exact_circular(n, shift):
    rng = np.random.default_rng(n)
    tx = rng.integers(0, 2, n, dtype=np.uint8)
    rx = np.roll(tx, shift) ^ (rng.random(n) < 0.1).astype(np.uint8)
    assert _xcorr(rx, tx, True) == _expected(rx, tx, True)


def test_bit_xcorr_uncorrelated_sidelobes_exact():
    rng = np.random.default_rng(3)
    rx = rng.integers(0, 2, 30000, dtype=np.uint8)
    tx = rng.integers(0, 2, 40000, dtype=np.uint8)
    assert _xcorr(rx, tx, False) == _expected(rx, tx, False)


@pytest.mark.parametrize("n_rx,n_tx,lag", [(50000, 1 << 16, 4321), (1 << 16, 70000, -999), (1 << 15, 1 << 15, 0)])
def test_frame_sync_device_equals_reference_formula(n_rx, n_tx, lag):
    rng = np.random.default_rng(lag & 0xFFFF)
    rx, tx = _streams(rng, n_rx, n_tx, lag, flip=0.02)
    if n_rx == n_tx:
        rx = np.roll(tx, 1000) ^ (rng.random(n_tx) < 0.02).astype(np.uint8)
    lag_h, a_h, b_h = frame_sync(rx, tx)
    dev = torch.device("cuda:0")
    lag_d, a_d, b_d = frame_sync_device(torch.from_numpy(rx).to(dev), torch.from_numpy(tx).to(dev))
    assert lag_d == lag_h
    assert np.array_equal(a_d.cpu().numpy(), a_h) and np.array_equal(b_d.cpu().numpy(), b_h)


def test_frame_sync_device_failure():
    rng = np.random.default_rng(9)
    rx = rng.integers(0, 2, 40000, dtype=np.uint8)
    tx = rng.integers(0, 2, 1 << 15, dtype=np.uint8)
    dev = torch.device("cuda:0")
    with pytest.raises(SyncFailure):
        frame_sync(rx, tx)
    with pytest.raises(SyncFailure):
        frame_sync_device(torch.from_numpy(rx).to(dev), torch.from_numpy(tx).to(dev))


def test_bit_xcorr_large_known_alignment():
    """2^27-bit streams (FFT 2^28 points, three passes): the peak lands on the
    inserted alignment with the exact overlap-minus-flips magnitude."""
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(5)
    n_tx = 1 << 27
    lag = 12_345_678
    n_rx = n_tx - lag - 1000
    tx = torch.randint(0, 2, (n_tx,), dtype=torch.uint8, device=dev, generator=g)
    flips = (torch.rand(n_rx, device=dev, generator=g) < 0.01).to(torch.uint8)
    rx = tx[lag:lag + n_rx] ^ flips
    nf = int(flips.sum())
    lag_d, a, b = frame_sync_device(rx, tx)
    assert lag_d == lag
    nws = int(_lib.load().kk_bit_xcorr_workspace_bytes(n_rx, n_tx, 0))
    ws = torch.empty(nws, dtype=torch.uint8, device=dev)
    out = torch.empty(3, dtype=torch.int64, device=dev)
    _lib.call("kk_bit_xcorr", rx.data_ptr(), n_rx, tx.data_ptr(), n_tx, 0, ws.data_ptr(), nws, out.data_ptr(),
              torch.cuda.current_stream().cuda_stream)
    k, peak, side = (int(v) for v in out.cpu())
    assert k == n_tx - 1 - lag and peak == n_rx - 2 * nf and side < peak // 100


def test_label_bits_error_windows_evm():
    from paper_2108_07001_b200.constellation import slicer_tables

    dev = torch.device("cuda:0")
    rng = np.random.default_rng(11)
    for order, k in ((4, 2), (16, 4), (64, 6)):
        pl = np.ascontiguousarray(slicer_tables(order).point_label, dtype=np.uint8)
        lab = rng.integers(0, order, 100_003, dtype=np.uint8)
        out = torch.empty(len(lab) * k, dtype=torch.uint8, device=dev)
        _lib.call("kk_label_bits", torch.from_numpy(lab).to(dev).data_ptr(), len(lab), pl.ctypes.data, order, k,
                  out.data_ptr(), torch.cuda.current_stream().cuda_stream)
        want = ((pl[lab][:, None] >> np.arange(k - 1, -1, -1)[None, :]) & 1).astype(np.uint8).reshape(-1)
        assert np.array_equal(out.cpu().numpy(), want)
    n = 1_000_003
    a = rng.integers(0, 2, n, dtype=np.uint8)
    b = a ^ (rng.random(n) < 0.003).astype(np.uint8)
    da, db = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    for bpw in (1, 7, 32, 1000, 65536, n):
        nw = n // bpw
        cnt = torch.zeros(1 + nw, dtype=torch.int64, device=dev)
        _lib.call("kk_bit_error_windows", da.data_ptr(), db.data_ptr(), n, bpw, cnt.data_ptr(), cnt[1:].data_ptr(),
                  torch.cuda.current_stream().cuda_stream)
        c = cnt.cpu().numpy()
        e = (a != b)
        assert c[0] == int(e.sum())
        assert np.array_equal(c[1:], e[: nw * bpw].reshape(nw, bpw).sum(1))
    s = (rng.standard_normal(50_001) + 1j * rng.standard_normal(50_001)).astype(np.complex64)
    r = rng.standard_normal(50_001) + 1j * rng.standard_normal(50_001)
    sums = torch.zeros(2 + 1024, dtype=torch.float64, device=dev)
    ds, dr = torch.from_numpy(s).to(dev), torch.from_numpy(r).to(dev)
    _lib.call("kk_evm_sums", ds.data_ptr(), dr.data_ptr(), len(s), sums.data_ptr(), sums[2:].data_ptr(),
              torch.cuda.current_stream().cuda_stream)
    se, sr = sums[:2].cpu().numpy()
    again = torch.zeros(2 + 1024, dtype=torch.float64, device=dev)
    _lib.call("kk_evm_sums", ds.data_ptr(), dr.data_ptr(), len(s), again.data_ptr(), again[2:].data_ptr(),
              torch.cuda.current_stream().cuda_stream)
    assert torch.equal(again[:2], sums[:2])   # deterministic
    assert abs(se - np.sum(np.abs(s.astype(np.complex128) - r) ** 2)) < 1e-9 * se
    assert abs(sr - np.sum(np.abs(r) ** 2)) < 1e-9 * sr


def test_measure_point_device_windowed_q():
    """windowed Q with windows much shorter than the stream: per-window
    counts from kk_bit_error_windows equal the reference formula's."""
    from types import SimpleNamespace

    from paper_2108_07001_b200.constellation import make_constellation
    from paper_2108_07001_b200.harness import measure_point, measure_point_device

    rng = np.random.default_rng(21)
    n = 300_000
    spec = make_constellation(16)
    idx = rng.integers(0, 16, n)
    syms = spec.points[idx]
    from paper_2108_07001_b200.constellation import slicer_tables
    pl = slicer_tables(16).point_label
    bits = ((pl[idx][:, None] >> np.arange(3, -1, -1)[None, :]) & 1).astype(np.uint8).reshape(-1)
    lab = idx.copy()
    err = rng.random(n) < 2e-3
    lab[err] = rng.integers(0, 16, int(err.sum()))
    soft = (syms + 0.05 * (rng.standard_normal(n) + 1j * rng.standard_normal(n))).astype(np.complex64)
    cfgx = SimpleNamespace(tx=SimpleNamespace(constellation_order=16, baud_hz=1e9),
                           rx=SimpleNamespace(startup_symbols=1000),
                           metrics=SimpleNamespace(head_guard_symbols=500, tail_guard_symbols=700,
                                                   windowed_q_window_s=20e-6))
    dev = torch.device("cuda:0")
    got = measure_point_device(torch.from_numpy(lab.astype(np.uint8)).to(dev), torch.from_numpy(soft).to(dev),
                               bits, syms, cfgx)
    want = measure_point(spec.points[lab], soft.astype(np.complex128), bits, syms, cfgx)
    assert len(want["windowed_q"]) > 5
    for key in ("n_bits", "n_errors", "sync_offset", "windowed_q"):
        assert got[key] == want[key], key
    assert abs(got["evm_pct"] - want["evm_pct"]) < 1e-9 * want["evm_pct"]


def test_bit_xcorr_minimum_sizes_and_errors():
    """Edge sizes of frame_sync (me:69-112): the shortest reference (2^14
    bits) against the shortest received stream (64 bits), and the errors the
    reference raises."""
    from paper_2108_07001_b200.sigcore import ParameterError

    rng = np.random.default_rng(17)
    tx = rng.integers(0, 2, 1 << 14, dtype=np.uint8)
    rx = tx[5000:5064].copy()
    assert _xcorr(rx, tx, False) == _expected(rx, tx, False)
    dev = torch.device("cuda:0")
    with pytest.raises(SyncFailure):
        frame_sync_device(torch.from_numpy(rx[:63]).to(dev), torch.from_numpy(tx).to(dev))
    with pytest.raises(ParameterError):
        frame_sync_device(torch.from_numpy(rx).to(dev), torch.from_numpy(tx[:(1 << 14) - 1]).to(dev))


def test_bit_xcorr_all_equal_streams():
    """Degenerate input: constant streams (every lag correlates) -- the peak
    is the full-overlap lag, the sidelobes are exact."""
    tx = np.ones(1 << 14, dtype=np.uint8)
    rx = np.ones(3000, dtype=np.uint8)
    assert _xcorr(rx, tx, False) == _expected(rx, tx, False)
