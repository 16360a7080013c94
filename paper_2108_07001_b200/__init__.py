"""paper_2108_07001_b200 -- B200-native (sm_100a) drop-in for the streaming
Kramers-Kronig receiver of arXiv 2108.07001 (reference package `kkmodem`).

Public surface mirrors kkmodem.rxdsp (see rxdsp.py); the per-sample work runs
in libkkb200.so (include/kkb200.h).  `harness` holds the device-resident
measurement helpers (BER, streaming bench) and `superframe` the multi-GPU
super-frame sharding.
"""

from .sigcore import (  # noqa: F401
    AdcCodes, AdcPacked12, BlockPlan, ComplexSignal, FirFilter, ParameterError, RealSignal,
    anti_alias_window, fir_frequency_response, pack12, read_adc_raw, unpack12, write_adc_raw,
)
from .constellation import ConstellationSpec, make_constellation  # noqa: F401
from .rxdsp import (  # noqa: F401
    DdlmsConfig, EqualizerState, GpuOptions, RxPipeline, RxPipelineConfig, SyncError,
    compute_static_taps, ddlms_wl, demap, design_receive_taps, downshift_dc, kk_reconstruct,
    refine_static_taps, static_equalize_and_resample, static_tap_coverage, stream_buffers,
    symbol_sync,
)

__version__ = "0.1.0"
