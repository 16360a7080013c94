"""Multi-GPU super-frame receive: one rank per GPU (torch.distributed, NCCL).

Everything before the DDLMS is local to a rank (superframe.py explains the
halos).  The DDLMS is one sequential recurrence across the whole stream
(rxdsp.py:465-498); ranks chain their frames exactly with the frame maps of
the phased solver (kk_ddlms_create/train/speculate/iterate/finish):

    rank 0 trains (exact) -> broadcast training-end taps T_te      (64 B)
    every rank speculates its frame from T_te -> frame map (P_r, Q_r)
    repeat:
        all_gather(P_r, Q_r)                                      (320 B/rank)
        T_start(r) = T_init . (P_0,Q_0) ... (P_{r-1},Q_{r-1})     (host, fp64)
        changed_r = iterate(T_start(r))  -> new (P_r, Q_r)
        all_reduce(sum changed)
    until no block of any rank changed its decisions.

At the fixpoint every rank's start taps are those of the sequential
recurrence, so the union of the ranks' decisions equals the single-stream
result.  The protocol (`solve_chained`) only needs a solver object and a
communicator, so tests/test_multirank_cpu.py runs it on CPU with gloo and a
float64 numpy solver double.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .constellation import slicer_tables
from .rxdsp import _T_from_wg, EqualizerState, RxPipeline, SyncError, _device, _ptr, _stream, _sync_device
from .superframe import SuperframeJob, SuperframeResult

MAP_LEN = 80   # P (8x8) + Q (2x8)


def compose_start(T_init: np.ndarray, maps: np.ndarray, rank: int) -> np.ndarray:
    """Exact start taps of `rank`'s frame: fold the frame maps of ranks
    0..rank-1 over the stream's initial taps (float64)."""
    T = np.asarray(T_init, np.float64).reshape(2, 8)
    for r in range(rank):
        P = np.asarray(maps[r][:64], np.float64).reshape(8, 8)
        Q = np.asarray(maps[r][64:], np.float64).reshape(2, 8)
        T = T @ P + Q
    return T.reshape(16).astype(np.float32)


class TorchComm:
    """The three collectives the protocol needs, on torch.distributed."""

    def __init__(self, dist, device):
        self.dist = dist
        # NCCL collectives take device tensors, gloo host tensors
        self.device = device if dist.get_backend() == "nccl" else "cpu"
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()

    def _t(self, a):
        import torch
        return torch.as_tensor(np.asarray(a, np.float64), device=self.device)

    def broadcast(self, a, src=0):
        t = self._t(a)
        self.dist.broadcast(t, src=src)
        return t.cpu().numpy()

    def all_gather(self, a):
        t = self._t(a)
        out = [t.clone() for _ in range(self.world)]
        self.dist.all_gather(out, t)
        return np.stack([o.cpu().numpy() for o in out])

    def all_reduce_sum(self, v):
        t = self._t([v])
        self.dist.all_reduce(t)
        return float(t.cpu().numpy()[0])


def solve_chained(solver, comm, T_init, has_training: bool, max_iter: int = 64):
    """The cross-rank exact DDLMS fixpoint; returns (iterations, stats)."""
    rank = comm.rank
    T_init = np.asarray(T_init, np.float32)
    if rank == 0 and has_training:
        T_te = solver.train(T_init)
    else:
        if rank == 0:
            solver.train(T_init)
        T_te = T_init
    T_te = comm.broadcast(T_te, src=0).astype(np.float32)
    mp = solver.speculate(T_te)
    per_iter = []
    soft_pass = False    # decision passes until no rank changed, then one soft refresh
    for it in range(1, max_iter + 1):
        maps = comm.all_gather(mp)
        T_start = compose_start(T_init, maps, rank)
        changed, rerun, mp = solver.iterate(T_start, soft_pass)
        total = comm.all_reduce_sum(changed)
        per_iter.append((int(changed), int(rerun), int(total)))
        if total == 0 and soft_pass:
            # nothing changed: `maps` are the converged frame maps
            solver.final_maps = maps
            return it, per_iter
        soft_pass = total == 0
    raise RuntimeError("multi-rank DDLMS did not converge within max_iter")


def guard_chain(comm, guard_counts, T_init, run_sequential):
    """Exact fallback when the divergence guard (rx:484-490) fired in some
    rank's frame: the affine maps assume unfrozen taps, so from the first
    rank r* whose frame saw a guard exceedance on, the recurrence is re-run
    in rank order with the exact sequential chain, each rank starting from
    the previous rank's end state (taps, frozen, div_count), broadcast.
    Ranks before r* had no exceedance: their frames and maps are exact, so
    r*'s start taps are the composition of their maps.  run_sequential(T,
    frozen, div_count) -> (T_end, frozen, div_count) re-runs this rank's
    frame.  Returns True when this rank's outputs were recomputed."""
    rank, world = comm.rank, comm.world
    first = next((r for r in range(world) if guard_counts[r] > 0), None)
    if first is None:
        return False
    state = np.zeros(18)
    if rank == first:
        state[:16] = compose_start(T_init, comm_maps(comm), first)
    state = comm.broadcast(state, src=first)
    for r in range(first, world):
        if rank == r:
            T, fz, dc = run_sequential(state[:16].astype(np.float32), bool(state[16]), int(state[17]))
            state[:16], state[16], state[17] = T, float(fz), float(dc)
        state = comm.broadcast(state, src=r)
    return rank >= first


def comm_maps(comm):
    return getattr(comm, "final_maps", None)


class GpuFrameSolver:
    """ctypes wrapper of the phased C solver over one device-resident frame."""

    def __init__(self, x_ptr, nsym, scale, train_ptr, n_train, cfg, dev):
        import torch

        d = cfg.ddlms
        tb = slicer_tables(cfg.constellation_order)
        self.tb = tb
        self.nsym = int(nsym)
        self.dev = dev
        B = int(cfg.gpu.ddlms_block)
        wsb = int(_lib.load().kk_ddlms_workspace_bytes(self.nsym, B))
        self.ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
        self.h = _lib.load().kk_ddlms_create(
            x_ptr, self.nsym, float(scale), train_ptr, int(n_train), tb.order, tb.pts_ri.ctypes.data,
            tb.grid.ctypes.data if tb.grid_m else None, tb.grid_m, tb.norm, tb.max_radius,
            float(d.divergence_factor), float(d.mu), B, float(cfg.gpu.ddlms_soft_tol), _ptr(self.ws), wsb,
            _stream(dev))
        if not self.h:
            _lib.check(_lib.KK_ERR_PARAM, "kk_ddlms_create")
        # the final pass writes straight into these
        self.labels = torch.empty(self.nsym, dtype=torch.uint8, device=dev)
        self.soft = torch.empty(self.nsym, dtype=torch.complex64, device=dev)
        _lib.call("kk_ddlms_bind_outputs", self.h, _ptr(self.labels), _ptr(self.soft))

    def train(self, T):
        out = np.zeros(16, np.float32)
        T = np.ascontiguousarray(T, np.float32)
        _lib.call("kk_ddlms_train", self.h, T.ctypes.data, out.ctypes.data)
        return out

    def speculate(self, T):
        mp = np.zeros(MAP_LEN, np.float32)
        T = np.ascontiguousarray(T, np.float32)
        _lib.call("kk_ddlms_speculate", self.h, T.ctypes.data, mp.ctypes.data)
        return mp

    def iterate(self, T, soft_pass=False):
        mp = np.zeros(MAP_LEN, np.float32)
        ch = ctypes.c_int64(0)
        rr = ctypes.c_int64(0)
        T = np.ascontiguousarray(T, np.float32)
        _lib.call("kk_ddlms_iterate", self.h, T.ctypes.data, int(bool(soft_pass)), ctypes.byref(ch),
                  ctypes.byref(rr), mp.ctypes.data)
        return ch.value, rr.value, mp

    def finish(self):
        labels, soft = self.labels, self.soft
        Tf = np.zeros(16, np.float32)
        guard = ctypes.c_int64(0)
        _lib.call("kk_ddlms_finish", self.h, _ptr(labels), _ptr(soft), Tf.ctypes.data, ctypes.byref(guard))
        return labels, soft, Tf, guard.value

    def close(self):
        if self.h:
            _lib.load().kk_ddlms_destroy(self.h)
            self.h = None
        self.ws = None


def _front_end_host(pipe, adc, chunk_samples: int, flush: bool, dev) -> None:
    """Front end of a pinned-host shard, chunk by chunk: every chunk's H2D
    copy is queued up front on a side stream (into one device staging
    buffer), the front end of each chunk waits only for its own copy."""
    import torch

    from .rxdsp import side_stream
    from .sigcore import AdcCodes, AdcPacked12

    p12 = isinstance(adc, AdcPacked12)
    host = adc.data if p12 else adc.codes
    n = len(adc)

    def span(a, b):   # element range of samples [a, b) (bytes for the packed format)
        return (3 * a // 2, 3 * b // 2) if p12 else (a, b)

    comp = torch.cuda.current_stream(dev)
    copy = side_stream(dev, "h2d")
    staging = torch.empty(span(0, n)[1], dtype=torch.uint8 if p12 else torch.int16, device=dev)
    starts = list(range(0, n, chunk_samples))
    ready = [torch.cuda.Event() for _ in starts]
    copy.wait_stream(comp)
    with torch.cuda.stream(copy):
        for i, a in enumerate(starts):
            e0, e1 = span(a, min(a + chunk_samples, n))
            staging[e0:e1].copy_(host[e0:e1], non_blocking=True)
            ready[i].record(copy)
    pipe.expect(n, chunk_samples)
    for i, a in enumerate(starts):
        m = min(chunk_samples, n - a)
        comp.wait_event(ready[i])
        e0, e1 = span(a, a + m)
        chunk = (AdcPacked12(staging[e0:e1], adc.half_lsb, m, adc.sample_rate_hz) if p12
                 else AdcCodes(staging[e0:e1], adc.half_lsb, adc.sample_rate_hz))
        pipe.front_end(chunk, flush=flush and i == len(starts) - 1)
    staging.record_stream(comp)


def receive_rank(cfg, adc, reference_prefix, job: SuperframeJob, dist, chunk_samples: int | None = None
                 ) -> SuperframeResult:
    """Receive this rank's super-frame of a multi-GPU stream."""
    import torch

    from .sigcore import AdcCodes, AdcPacked12

    dev = _device()
    comm = TorchComm(dist, dev)
    hop = cfg.static_plan.hop
    pipe = RxPipeline(cfg, reference_symbols=reference_prefix if job.rank == 0 else None,
                      stream_offset=job.load_start, static_start_hop=job.core_start // hop)
    host_t = adc.data if isinstance(adc, AdcPacked12) else (adc.codes if isinstance(adc, AdcCodes) else None)
    if chunk_samples and isinstance(host_t, torch.Tensor) and not host_t.is_cuda:
        _front_end_host(pipe, adc, int(chunk_samples), job.last, dev)
    else:
        pipe.front_end(adc, flush=job.last)
    # ---- sync + eq scale on rank 0 (stream head), broadcast ----
    info = np.zeros(4)
    if job.rank == 0:
        need = cfg.sync_wait_samples + 2 * cfg.sync_symbols
        nh = min(need, pipe._y2.end)
        head = pipe._y2.view(0, nh)
        ref = pipe._ref_dev[:cfg.sync_symbols] if pipe._ref_dev is not None else None
        parity, k, ratio, rms = _sync_device(head, ref, min(nh // 2, 1 << 13), dev)
        if ref is not None and (parity < 0 or ratio < 4.0):
            raise SyncError(f"no correlation peak (peak-to-rms {ratio:.2f})")
        offset = 2 * k + parity if ref is not None else 1
        info[:] = [offset, ratio, (1.0 / rms) if rms > 0 else 1.0, 0]
    info = comm.broadcast(info, src=0)
    offset, ratio, scale = int(info[0]), float(info[1]), float(info[2])
    drop = max(0, offset - 1) if reference_prefix is not None else 0
    # ---- this rank's DDLMS symbols [k0, k1) on the global symbol grid ----
    q0 = job.core_start // 2
    k0 = max(0, -(-(q0 - drop) // 2))
    if job.last:
        n_q = pipe._y2.end - drop
        k1 = (n_q - cfg.ddlms.n_taps) // 2 + 1
    else:
        k1 = max(0, -(-(job.core_end // 2 - drop) // 2))
    nsym = k1 - k0
    train_total = min(cfg.ddlms.startup_symbols, len(reference_prefix)) if reference_prefix is not None else 0
    n_train = int(max(0, min(nsym, train_total - k0)))
    train_ptr = (pipe._ref_dev.data_ptr() + k0 * 8) if (n_train > 0 and pipe._ref_dev is not None) else 0
    t_dd0 = pipe._ev()          # the chained DDLMS counts as the "ddlms" stage (rx:652-654)
    solver = GpuFrameSolver(pipe._y2.ptr(drop + 2 * k0), nsym, scale, train_ptr, n_train, cfg, dev)
    st0 = EqualizerState.initial(cfg.ddlms.n_taps)
    T_init = _T_from_wg(st0.w, st0.g)
    iters, per_iter = solve_chained(solver, comm, T_init, has_training=n_train > 0,
                                    max_iter=int(cfg.gpu.ddlms_max_iter))
    labels, soft, _, guard = solver.finish()
    comm.final_maps = solver.final_maps
    solver.close()
    mode = "multirank"
    guards = comm.all_gather([float(guard)])[:, 0]

    def run_sequential(T, frozen, div_count):
        import torch

        from .rxdsp import _seq_ddlms, _wg_from_T

        w, g = _wg_from_T(T)
        wg = torch.from_numpy(np.concatenate([w, g]).astype(np.complex64)).to(dev)
        fz = torch.tensor([int(frozen), int(div_count)], dtype=torch.int32, device=dev)
        tv = pipe._ref_dev[k0:k0 + n_train] if n_train > 0 else None
        xv = pipe._y2.view(drop + 2 * k0, drop + 2 * k0 + 2 * nsym + 2)
        _seq_ddlms(xv, nsym, scale, cfg.ddlms, solver.tb.order, wg, fz, tv, n_train, labels, soft, None, dev)
        wgh = wg.cpu().numpy().astype(np.complex128)
        f = fz.cpu().numpy()
        return _T_from_wg(wgh[:4], wgh[4:]), bool(f[0]), int(f[1])

    if guard_chain(comm, guards, T_init, run_sequential):
        mode = "multirank(guard: sequential chain)"
    pipe._events.append(("ddlms", t_dd0, pipe._ev()))
    pipe.release_buffers()
    stats = [{"k0": k0, "nsym": nsym, "mode": mode, "iterations": iters, "per_iter": per_iter}]
    return SuperframeResult(labels, soft, k0, pipe, stats, offset if job.rank == 0 else None)
