"""Super-frame sharding of one ADC stream across GPUs.

Rank r of W owns ADC samples [r*L, (r+1)*L) of a continuous W*L-sample
stream.  Everything up to the DDLMS is local and exact on the global grids
(KK hops of 512, carrier segments of 65536, static hops of 16384, downshift
phase (p*g mod q)): a rank loads a left halo of HALO_SAMPLES (two carrier
segments -- the first absorbs the KK state warm-up, the second gives exact
carrier means and the static overlap) and a right halo of one carrier
segment (the last symbols' 4-tap windows reach 3 samples past the core).
Rank 0 alone sees the stream head: it computes the sync offset / eq scale
and the training-end taps and broadcasts them.  The DDLMS is one sequential
recurrence across ranks; it is solved exactly with the affine fixpoint of
kk_ddlms_solve lifted one level up: per iteration every rank all-gathers
the composed map (P_r, Q_r) of its frame (64 + 16 floats), composes the
exclusive prefix of the ranks before it to get its exact start taps, re-runs
its blocks and all-reduces the changed-decision count.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

HALO_SAMPLES = 2 * 65536
RIGHT_HALO_SAMPLES = 65536


@dataclass
class SuperframeJob:
    rank: int
    world: int
    core_start: int
    core_end: int
    load_start: int
    load_end: int

    @property
    def last(self) -> bool:
        return self.rank == self.world - 1


def plan_superframe(rank: int, world: int, samples_per_rank: int, halo: int = HALO_SAMPLES,
                    right_halo: int = RIGHT_HALO_SAMPLES) -> SuperframeJob:
    if samples_per_rank % 65536:
        raise ValueError("super-frames must be whole carrier segments (65536 samples)")
    cs, ce = rank * samples_per_rank, (rank + 1) * samples_per_rank
    ls = max(0, cs - halo)
    le = ce if rank == world - 1 else ce + right_halo
    return SuperframeJob(rank, world, cs, ce, ls, le)


@dataclass
class SuperframeResult:
    labels: object              # uint8 device tensor: point index per owned symbol (255 = training)
    soft: object                # complex64 device tensor
    first_symbol: int           # global DDLMS symbol index of labels[0]
    pipe: object = None         # the pipeline (stage timing events resolved lazily)
    stats: list | None = None   # explicit per-frame statistics (multi-rank); else the pipeline's
    sync_offset: int | None = None

    @property
    def stage_seconds(self) -> dict:
        return self.pipe.stage_seconds if self.pipe is not None else {}

    @property
    def ddlms_stats(self) -> list:
        """Per-frame DDLMS statistics (materialised on first access: the
        single-rank solve is asynchronous)."""
        if self.stats is not None:
            return self.stats
        return self.pipe.ddlms_stats if self.pipe is not None else []


def receive_superframe(cfg, adc, reference_prefix, job: SuperframeJob, dist=None,
                       chunk_samples: int | None = None) -> SuperframeResult:
    """Receive this rank's super-frame.  adc: AdcCodes / ndarray / CUDA tensor
    covering [job.load_start, job.load_end).  Multi-rank with AdcCodes over a
    pinned HOST tensor and chunk_samples: the shard is ingested chunk by chunk
    (H2D copies overlapped with the front end)."""
    from .rxdsp import RxPipeline

    if job.world == 1:
        pipe = RxPipeline(cfg, reference_symbols=reference_prefix)
        pipe.feed(adc, flush=True)
        labels, soft, meta = pipe.drain_device()
        pipe.release_buffers()
        return SuperframeResult(labels, soft, meta[0][0] if meta else 0, pipe, None, pipe.sync_offset)
    from .multirank import receive_rank
    return receive_rank(cfg, adc, reference_prefix, job, dist, chunk_samples=chunk_samples)
