"""CPU checks (numpy, float64) of the algebra every CUDA kernel relies on,
against the oracle restatement of the reference:

* K1: two real KK blocks packed as one complex 1024-FFT with the Hermitian
  extension of the reference's rfft multiplier (rxdsp.py:170-181, :227-230);
* K2: the 32768-point block never materialised -- radix-2 DIF split into
  even/odd 16384-FFTs, kept quarters, two 8192-IFFTs and the final combine
  (rxdsp.py:714-720);
* the in-place Stockham pass index math (mixed radix) and the padded float2
  shared-memory layout being bank-conflict free for every access pattern;
* the two-level twiddle tables and running-product twiddle chains;
* DDLMS: the real 2x8 form of the widely-linear recurrence, the per-block
  affine maps (P_b, Q_b = T_end - T_start P_b), and the speculative affine
  prefix-scan fixpoint reproducing the sequential decisions exactly
  (rxdsp.py:460-499).
"""

import numpy as np
import pytest

from oracle import kkoracle as ko
from paper_2108_07001_b200.rxdsp import _T_from_wg, _tone_rotation, _wg_from_T

rng = np.random.default_rng(0)


def stockham(x, radices, inverse=False):
    N = len(x)
    data = x.astype(np.complex128).copy()
    sign = 1 if inverse else -1
    Ns = 1
    for R in radices:
        out = np.empty_like(data)
        for j in range(N // R):
            v = np.array([data[j + r * N // R] for r in range(R)])
            v = v * np.exp(sign * 2j * np.pi * (j % Ns) * np.arange(R) / (Ns * R))
            v = np.fft.fft(v) if not inverse else np.fft.ifft(v) * R
            d0 = (j // Ns) * Ns * R + (j % Ns)
            for r in range(R):
                out[d0 + r * Ns] = v[r]
        data = out
        Ns *= R
    return data


@pytest.mark.parametrize("N,rad", [(1024, [16, 16, 4]), (16384, [16, 16, 16, 4]), (8192, [16, 16, 8, 4])])
def test_stockham_plans(N, rad):
    x = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    assert np.max(np.abs(stockham(x, rad) - np.fft.fft(x))) < 1e-9
    assert np.max(np.abs(stockham(x, rad, True) - np.fft.ifft(x) * N)) < 1e-9


def padi(i):
    return i + (i >> 4)


@pytest.mark.parametrize("N,rad,NT", [(16384, [16, 16, 16, 4], 512), (8192, [16, 16, 8, 4], 512),
                                      (1024, [16, 16, 4], 64)])
def test_padded_layout_conflict_free(N, rad, NT):
    """Every LDS.64/STS.64 half-warp (16 lanes) of every pass hits 16
    distinct bank pairs under padi(i) = i + i/16."""
    Ns = 1
    for R in rad:
        NB = N // R
        for q in range(max(1, NB // NT)):
            for w0 in range(0, min(NT, NB), 16):
                js = np.arange(w0, w0 + 16) + q * NT
                for r in range(R):
                    rd = padi(js + r * NB) % 16
                    d0 = (js // Ns) * Ns * R + js % Ns
                    wr = padi(d0 + r * Ns) % 16
                    assert len(set(rd)) == 16 and len(set(wr)) == 16
        Ns *= R


def test_k1_pair_packing():
    nfft = 1024
    mult = ko.hilbert_mult(nfft, 256)
    ua, ub = rng.standard_normal(nfft), rng.standard_normal(nfft)
    pa = np.fft.irfft(np.fft.rfft(ua) * mult, n=nfft)
    pb = np.fft.irfft(np.fft.rfft(ub) * mult, n=nfft)
    k = np.arange(nfft)
    M = np.zeros(nfft, complex)
    lo = (k >= 1) & (k <= 511)
    M[lo] = (-1j) ** ((k[lo] + 1) % 4)
    hi = k >= 513
    M[hi] = np.conj((-1j) ** ((1025 - k[hi]) % 4))
    assert np.max(np.abs(M[:513] - mult)) < 1e-12
    z = np.fft.ifft(np.fft.fft(ua + 1j * ub) * M)
    assert np.max(np.abs(z.real - pa)) < 1e-12 and np.max(np.abs(z.imag - pb)) < 1e-12


def test_k2_even_odd_split_matches_reference_static():
    n, m = 32768, 16384
    taps = rng.standard_normal(203) + 1j * rng.standard_normal(203)
    kept, H = ko.static_response(taps, 2e9, n, 4e9, 0.01, n // 4)
    blk = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    ref = (np.fft.ifft(np.fft.fft(blk)[kept] * H) * (m / n))[m // 2:]
    x0, x1 = blk[:m], blk[m:]
    E = np.fft.fft(x0 + x1)
    O = np.fft.fft((x0 - x1) * np.exp(-2j * np.pi * np.arange(m) / n))
    mp = np.arange(8192)
    src = np.where(mp < 4096, mp, mp + 8192)
    A = np.fft.ifft(E[src] * H[0::2]) * 8192
    B = np.fft.ifft(O[src] * H[1::2]) * 8192
    r = np.arange(8192)
    out = (A - np.exp(2j * np.pi * r / 16384) * B) * (0.5 / 16384)
    assert np.max(np.abs(out - ref)) < 1e-12 * np.max(np.abs(ref))


def test_twiddle_tables_and_chains():
    for M in (256, 1024, 2048, 4096, 8192, 16384, 32768):
        L = np.exp(-2j * np.pi * np.arange(32) / M).astype(np.complex64)
        H = np.exp(-2j * np.pi * 32 * np.arange(M // 32) / M).astype(np.complex64)
        k = np.arange(M)
        w = (H[k >> 5].astype(np.complex128) * L[k & 31])
        assert np.max(np.abs(w - np.exp(-2j * np.pi * k / M))) < 2e-7
    # running product w1^r, r < 16, in float32
    w1 = np.complex64(np.exp(-2j * np.pi * 37 / 4096))
    wr, worst = w1, 0.0
    for r in range(1, 16):
        worst = max(worst, abs(complex(wr) - np.exp(-2j * np.pi * 37 * r / 4096)))
        wr = np.complex64(wr * w1)
    assert worst < 2e-6


def test_tone_rotation_is_exact_rational():
    p, q, tab, step = _tone_rotation(0.516e9, 4e9)
    assert (p, q, step) == (129, 1000, 0)
    n = np.array([0, 1, 999, 1000, 2 ** 30 + 12345, 2 ** 40 + 7])
    exact = np.exp(-2j * np.pi * ((p * (n % q)) % q) / q)
    assert np.max(np.abs(tab[(p * (n % q)) % q] - exact)) < 1e-7


@pytest.mark.parametrize("tone", [0.5123456789e9, 0.516e9 + 1.0, -0.3e9 + 0.123, 1.2345e9])
def test_tone_rotation_general_fixed_point(tone):
    """Tones that are not p/q with q <= 1024: a 64-bit fixed-point phase step
    (K1/K2 compute exp(-2 pi i (g step mod 2^64) / 2^64)); the phase equals
    the float64 phase of sigcore.py frequency_shift :297-298 to ~1e-7 rad at
    g ~ 2^30 (the float64 reference's own rounding)."""
    from fractions import Fraction

    p, q, tab, step = _tone_rotation(tone, 4e9)
    assert q == 0 and tab is None and 0 < step < 2 ** 64
    for g in (0, 1, 12345, 2 ** 30 + 777, 2 ** 36 + 5):
        ph = (g * step) % 2 ** 64
        cyc = ph / 2 ** 64
        exact = (Fraction(tone) / Fraction(4e9) * g) % 1
        d = abs(cyc - float(exact))
        assert min(d, 1 - d) * 2 * np.pi < 1e-9 * max(1, g / 2 ** 20)


def test_wl_taps_real_form_roundtrip():
    w = rng.standard_normal(4) + 1j * rng.standard_normal(4)
    g = rng.standard_normal(4) + 1j * rng.standard_normal(4)
    w2, g2 = _wg_from_T(_T_from_wg(w, g))
    assert np.max(np.abs(w2 - w)) < 1e-6 and np.max(np.abs(g2 - g)) < 1e-6


# ---------------------------------------------------------------------------
# DDLMS: real form, block maps, speculative affine scan (numpy model of
# kk_ddlms_solve, float64) -- must reproduce the sequential oracle exactly
# ---------------------------------------------------------------------------

def T_from_wg64(w, g):
    T = np.zeros((2, 8))
    T[0, 0::2] = w.real + g.real
    T[0, 1::2] = w.imag - g.imag
    T[1, 0::2] = -w.imag - g.imag
    T[1, 1::2] = w.real - g.real
    return T


def windows(x, n):
    X = np.empty((n, 8))
    for u in range(4):
        X[:, 2 * u] = x[u:u + 2 * n:2].real
        X[:, 2 * u + 1] = x[u:u + 2 * n:2].imag
    return X


def run_block(T, X, D_train, pts, mu):
    """Sequential real-form run of one block; returns labels, soft, end taps."""
    T = T.copy()
    labs, soft = [], []
    for k in range(len(X)):
        y = T @ X[k]
        if k < len(D_train):
            d, lab = D_train[k], 255
        else:
            lab = int(np.argmin(np.abs((y[0] + 1j * y[1]) - pts)))
            d = pts[lab]
        T = T + 2 * mu * np.outer([d.real - y[0], d.imag - y[1]], X[k])
        labs.append(lab)
        soft.append(y[0] + 1j * y[1])
    return np.array(labs), np.array(soft), T


def spec_scan_solve(x, train, pts, mu, B, T0):
    n = (len(x) - 4) // 2 + 1
    X = windows(x, n)
    nb = -(-n // B)
    blocks = [(b * B, min(n, (b + 1) * B)) for b in range(nb)]
    P = []
    for k0, k1 in blocks:
        Pm = np.eye(8)
        for k in range(k0, k1):
            Pm = Pm @ (np.eye(8) - 2 * mu * np.outer(X[k], X[k]))
        P.append(Pm)
    labels = np.full(n, -1)
    soft = np.zeros(n, complex)
    Q = [None] * nb
    Tstart = [T0.copy() for _ in range(nb)]
    # training blocks exact from any start, then speculate from the training end
    bt = min(len(train) // B, nb)
    for b in range(bt):
        k0, k1 = blocks[b]
        lab, sf, Te = run_block(T0, X[k0:k1], train[k0:k1], pts, mu)
        Q[b] = Te - T0 @ P[b]
    Tg = T0.copy()
    for b in range(bt):
        Tg = Tg @ P[b] + Q[b]
    iters = 0
    for b in range(nb):
        Tstart[b] = T0 if b == 0 else (Tg if b >= bt else Tstart[b])
    for it in range(nb + 1):
        # re-run every block from its current start; count changes
        changed = 0
        for b in range(nb):
            k0, k1 = blocks[b]
            lab, sf, Te = run_block(Tstart[b], X[k0:k1], train[k0:min(k1, len(train))], pts, mu)
            if not np.array_equal(lab, labels[k0:k1]):
                changed += 1
            labels[k0:k1], soft[k0:k1] = lab, sf
            Q[b] = Te - Tstart[b] @ P[b]
        iters += 1
        if changed == 0:
            break
        # exclusive prefix scan of the affine maps
        T = T0.copy()
        for b in range(nb):
            Tstart[b] = T
            T = T @ P[b] + Q[b]
    return labels, soft, iters


@pytest.mark.parametrize("order,noise", [(16, 0.08), (64, 0.03)])
def test_speculative_scan_reproduces_sequential(order, noise):
    spec = ko.constellation(order)
    n_sym = 3000
    syms = spec.points[rng.integers(0, order, n_sym)]
    x = np.repeat(syms, 2) * (0.9 + 0.1j) + noise * (rng.standard_normal(2 * n_sym) + 1j * rng.standard_normal(2 * n_sym))
    x = 0.95 * x + 0.05 * np.conj(x)
    train = syms[:600]
    mu = 2e-3
    dec_ref, soft_ref, _ = ko.ddlms_wl(x, ko.EqState.initial(), training=train, order=order, mu=mu)
    lab_ref = ko.to_index(dec_ref, order)
    T0 = T_from_wg64(np.array([0, 1, 0, 0], complex), np.zeros(4, complex))
    labels, soft, iters = spec_scan_solve(x, train, spec.points, mu, 64, T0)
    dd = np.arange(len(labels)) >= len(train)
    assert np.array_equal(labels[dd], lab_ref[dd]), f"decisions differ after {iters} iterations"
    assert np.max(np.abs(soft - soft_ref)) < 1e-9
    assert iters >= 2
