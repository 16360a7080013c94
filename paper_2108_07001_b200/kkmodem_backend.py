"""Backend switch: run the reference package `kkmodem` on the B200 receiver.

This is the binding INTEGRATION.md §1 describes, packaged so it can be
applied without editing kkmodem:

    import paper_2108_07001_b200.kkmodem_backend as kb
    kb.install()            # after `import kkmodem`, before importing its callers

or, for the reference's own test-suite,

    python -m pytest -p paper_2108_07001_b200.kkmodem_backend <kkmodem tests>

`install()` rebinds the receive-path names of `kkmodem.rxdsp`
(rxdsp.py:608-824 `RxPipeline` and the functional stages rx:184-601) to this
package, the names `kkmodem.harness.runner` imported from it by value
(runner.py:16-24: `RxPipeline`, `demap`), and the nonlinear fiber span
`kkmodem.channel.ssfm_span` (channel.py:124-158, called by name from
propagate_link :208-209) to the GPU split-step span.
Everything else -- transmitter, linear channel, front end, metrics, sweeps,
CLI -- stays the reference's own code,
so `run_single`, `run_sweep`, `run_sustained` and `bench_throughput` drive
the GPU receiver unmodified.  The exception types this package raises are
subclasses of kkmodem's (`sigcore.ParameterError` sigcore.py:37,
`rxdsp.SyncError` rxdsp.py:63) whenever kkmodem is importable, so the
reference's `except SyncError` (runner.py:182) catches GPU sync failures.

Test modules bind names at import time (`from kkmodem.rxdsp import
RxPipeline`), so the switch must be installed before they are collected:
the pytest plugin hook below does that.
"""

from __future__ import annotations

# receive-path names rebound in kkmodem.rxdsp (rx:144-601 functional stages,
# rx:608-824 the pipeline); tap design (rx:264-394) is host setup and stays
# the reference's
RXDSP_NAMES = (
    "RxPipeline",
    "kk_reconstruct",
    "downshift_dc",
    "static_equalize_and_resample",
    "ddlms_wl",
    "demap",
    "symbol_sync",
)
# names harness/runner.py:16-24 imported by value from ..rxdsp
RUNNER_NAMES = ("RxPipeline", "demap")
# the nonlinear span of kkmodem.channel (propagate_link looks it up by name)
CHANNEL_NAMES = ("ssfm_span",)

_saved: dict | None = None


def installed() -> bool:
    return _saved is not None


def install() -> None:
    """Rebind kkmodem's receiver to the B200 implementation (idempotent)."""
    global _saved
    if _saved is not None:
        return
    import kkmodem.channel as kch
    import kkmodem.rxdsp as krx
    import kkmodem.harness.runner as krun

    from . import channel as gch
    from . import rxdsp as gpu
    from ._lib import SyncError
    from .sigcore import ParameterError

    import kkmodem.sigcore as ksc

    # the GPU exception types must be catchable as kkmodem's
    if not issubclass(SyncError, krx.SyncError) or not issubclass(ParameterError, ksc.ParameterError):
        raise RuntimeError(
            "paper_2108_07001_b200 was imported before kkmodem was importable: its exception types "
            "cannot subclass kkmodem's.  Put kkmodem on sys.path before importing paper_2108_07001_b200.")
    gpu._lib.load()
    saved = {("rx", n): getattr(krx, n) for n in RXDSP_NAMES}
    saved.update({("run", n): getattr(krun, n) for n in RUNNER_NAMES})
    saved.update({("ch", n): getattr(kch, n) for n in CHANNEL_NAMES})
    for n in RXDSP_NAMES:
        setattr(krx, n, getattr(gpu, n))
    for n in RUNNER_NAMES:
        setattr(krun, n, getattr(gpu, n))
    for n in CHANNEL_NAMES:
        setattr(kch, n, getattr(gch, n))
    _saved = saved


def uninstall() -> None:
    """Restore kkmodem's own receiver."""
    global _saved
    if _saved is None:
        return
    import kkmodem.channel as kch
    import kkmodem.rxdsp as krx
    import kkmodem.harness.runner as krun

    mods = {"rx": krx, "run": krun, "ch": kch}
    for (where, n), v in _saved.items():
        setattr(mods[where], n, v)
    _saved = None


# -- pytest plugin (-p paper_2108_07001_b200.kkmodem_backend) ---------------

def pytest_configure(config):  # noqa: D401 - pytest hook
    install()
    config.addinivalue_line("markers", "gpu: needs a CUDA device")


def pytest_report_header(config):
    return "kkmodem receiver backend: B200 (paper_2108_07001_b200, libkkb200.so)"
