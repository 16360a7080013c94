"""Multi-rank (world size 2) host logic on CPU with the gloo backend.

The cross-rank DDLMS protocol of paper_2108_07001_b200.multirank
(`solve_chained`: rank-0 training broadcast, per-iteration all_gather of
frame maps, exclusive-prefix composition, all_reduce of changed blocks) is
run with a float64 numpy stand-in for the GPU frame solver; the union of the
two ranks' decisions must equal the single-stream sequential recurrence of
the oracle (rxdsp.py:465-498) exactly.
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def windows(x, n):
    X = np.empty((n, 8))
    for u in range(4):
        X[:, 2 * u] = x[u:u + 2 * n:2].real
        X[:, 2 * u + 1] = x[u:u + 2 * n:2].imag
    return X


class NumpyFrameSolver:
    """float64 model of the phased GPU solver (kk_ddlms_create & co.)."""

    def __init__(self, X, train, pts, mu, B):
        self.X, self.train_syms, self.pts, self.mu, self.B = X, train, pts, mu, B
        n = len(X)
        self.blocks = [(b * B, min(n, (b + 1) * B)) for b in range(-(-n // B))]
        self.P = []
        for k0, k1 in self.blocks:
            Pm = np.eye(8)
            for k in range(k0, k1):
                Pm = Pm @ (np.eye(8) - 2 * mu * np.outer(X[k], X[k]))
            self.P.append(Pm)
        self.labels = np.full(n, -1)
        self.soft = np.zeros(n, complex)
        self.Q = [np.zeros((2, 8)) for _ in self.blocks]
        self.bt = min(len(train) // B, len(self.blocks))

    def _run(self, b, T):
        k0, k1 = self.blocks[b]
        T0 = T.copy()
        T = T.copy()
        labs = []
        for k in range(k0, k1):
            y = T @ self.X[k]
            if k < len(self.train_syms):
                d, lab = self.train_syms[k], 255
            else:
                lab = int(np.argmin(np.abs((y[0] + 1j * y[1]) - self.pts)))
                d = self.pts[lab]
            T = T + 2 * self.mu * np.outer([d.real - y[0], d.imag - y[1]], self.X[k])
            labs.append(lab)
            self.soft[k] = y[0] + 1j * y[1]
        changed = not np.array_equal(self.labels[k0:k1], labs)
        self.labels[k0:k1] = labs
        self.Q[b] = T - T0 @ self.P[b]
        return changed

    def _map(self):
        P, Q = np.eye(8), np.zeros((2, 8))
        for b in range(len(self.blocks)):
            P, Q = P @ self.P[b], Q @ self.P[b] + self.Q[b]
        return np.concatenate([P.reshape(-1), Q.reshape(-1)])

    def train(self, T):
        T = np.asarray(T, np.float64).reshape(2, 8)
        for b in range(self.bt):
            self._run(b, T)
        for b in range(self.bt):
            T = T @ self.P[b] + self.Q[b]
        return T.reshape(-1).astype(np.float32)

    def speculate(self, Tg):
        Tg = np.asarray(Tg, np.float64).reshape(2, 8)
        for b in range(self.bt, len(self.blocks)):
            self._run(b, Tg)
        return self._map()

    def iterate(self, Ts, soft_pass=False):
        T = np.asarray(Ts, np.float64).reshape(2, 8)
        changed = 0
        for b in range(len(self.blocks)):
            changed += self._run(b, T)
            T = T @ self.P[b] + self.Q[b]
        return changed, len(self.blocks), self._map()


def make_stream(seed=5, n_sym=4000, order=16):
    from oracle import kkoracle as ko

    rng = np.random.default_rng(seed)
    pts = ko.constellation(order).points
    syms = pts[rng.integers(0, order, n_sym)]
    x = np.repeat(syms, 2) * (0.9 + 0.1j) + 0.08 * (rng.standard_normal(2 * n_sym) + 1j * rng.standard_normal(2 * n_sym))
    return syms, 0.95 * x + 0.05 * np.conj(x), pts


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2108_07001_b200.multirank import TorchComm, solve_chained
        from paper_2108_07001_b200.rxdsp import EqualizerState, _T_from_wg

        syms, x, pts = make_stream()
        n = (len(x) - 4) // 2 + 1
        X = windows(x, n)
        n_train, mu, B = 700, 2e-3, 64
        cut = n // 2 + 37                      # rank boundary (global symbol grid)
        k0, k1 = (0, cut) if rank == 0 else (cut, n)
        train = syms[:n_train] if rank == 0 else np.zeros(0, complex)
        solver = NumpyFrameSolver(X[k0:k1], train, pts, mu, B)
        st0 = EqualizerState.initial()
        T_init = _T_from_wg(st0.w, st0.g).astype(np.float64)
        comm = TorchComm(dist, torch.device("cpu"))
        iters, per_iter = solve_chained(solver, comm, T_init, has_training=rank == 0)
        out_q.put((rank, k0, solver.labels.copy(), solver.soft.copy(), iters, per_iter))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_chained_ddlms_equals_sequential():
    from oracle import kkoracle as ko

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    labels = np.concatenate([r[2] for r in res])
    soft = np.concatenate([r[3] for r in res])
    syms, x, pts = make_stream()
    dec_ref, soft_ref, _ = ko.ddlms_wl(x, ko.EqState.initial(), training=syms[:700], order=16, mu=2e-3)
    lab_ref = ko.to_index(dec_ref, 16)
    dd = np.arange(len(labels)) >= 700
    assert np.array_equal(labels[dd], lab_ref[dd])
    # start taps cross ranks as float32 (as on the GPU): soft within 1e-6
    assert np.max(np.abs(soft - soft_ref)) < 1e-6
    assert res[0][4] == res[1][4] and res[0][4] >= 2      # same global iteration count


def _guard_worker(rank, world, port, out_q):
    """Rank 1's frame holds a burst that trips the divergence guard: the
    chained fallback must reproduce the single-stream recurrence (frozen
    taps and all) exactly."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import kkoracle as ko
        from paper_2108_07001_b200.multirank import TorchComm, guard_chain
        from paper_2108_07001_b200.rxdsp import EqualizerState, _T_from_wg, _wg_from_T

        syms, x, pts = make_guard_stream()
        n = (len(x) - 4) // 2 + 1
        cut = n // 2 + 37
        k0, k1 = (0, cut) if rank == 0 else (cut, n)
        st0 = EqualizerState.initial()
        T_init = _T_from_wg(st0.w, st0.g).astype(np.float64)
        comm = TorchComm(dist, torch.device("cpu"))
        # rank 0's converged frame map (exact: no guard there), as the
        # solver would have all-gathered it: the sequential oracle's end taps
        # from T_init over rank 0's symbols, written as P = I, Q = T_end - T_init
        st = ko.EqState.initial()
        ko.ddlms_wl(x[:2 * cut + 2], st, training=syms[:700], order=16, mu=2e-3)
        P = np.eye(8)
        Q = (_T_from_wg(st.w, st.g).astype(np.float64) - T_init).reshape(2, 8)
        comm.final_maps = np.stack([np.concatenate([P.ravel(), Q.ravel()])] * world)
        out = {}

        def run_sequential(T, frozen, div_count):
            w, g = _wg_from_T(T)
            s = ko.EqState(w=w.copy(), g=g.copy(), frozen=frozen, div_count=div_count)
            tr = syms[k0:700] if k0 < 700 else None
            dec, soft, s = ko.ddlms_wl(x[2 * k0:2 * k1 + 2], s, training=tr, order=16, mu=2e-3)
            out["labels"] = ko.to_index(dec[:k1 - k0], 16)
            return _T_from_wg(s.w, s.g), s.frozen, s.div_count

        guards = [0.0, 5.0]                           # rank 1 saw exceedances
        redone = guard_chain(comm, guards, T_init, run_sequential)
        out_q.put((rank, redone, out.get("labels")))
    finally:
        dist.destroy_process_group()


def make_guard_stream():
    syms, x, pts = make_stream(seed=9)
    n = len(syms)
    x = x.copy()
    x[2 * (3 * n // 4):2 * (3 * n // 4 + 150)] *= 40.0     # 150 symbols far outside 10 x max radius
    return syms, x, pts


def test_two_rank_guard_fallback_equals_sequential():
    from oracle import kkoracle as ko

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_guard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][1] is False and res[1][1] is True       # only rank 1 re-ran
    syms, x, pts = make_guard_stream()
    st = ko.EqState.initial()
    dec_ref, _, st = ko.ddlms_wl(x, st, training=syms[:700], order=16, mu=2e-3)
    assert st.frozen                                       # the burst did trip the guard
    n = len(dec_ref)
    cut = n // 2 + 37
    lab_ref = ko.to_index(dec_ref, 16)
    assert np.array_equal(res[1][2], lab_ref[cut:])
