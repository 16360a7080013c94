"""ctypes binding of libkkb200.so (the C ABI declared in include/kkb200.h).

There is no CPU fallback: if the CUDA library is missing or cannot be loaded
every entry point raises.  Status codes map onto the reference's exception
types (ParameterError sigcore.py:37, SyncError rxdsp.py:63, RuntimeError).
"""

from __future__ import annotations

import ctypes
import os

from .sigcore import ParameterError, kkmodem_class

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libkkb200.so")

KK_OK, KK_ERR_PARAM, KK_ERR_SYNC, KK_ERR_CUDA, KK_ERR_INTERNAL = 0, 1, 2, 3, 4
KK_DTYPE_I16, KK_DTYPE_F32, KK_DTYPE_F64, KK_DTYPE_P12 = 0, 1, 2, 3
KK_DTYPE_PRECISE = 0x100   # or-ed flag: correctly rounded transcendental functions


_KK_SYNC_ERROR = kkmodem_class("kkmodem.rxdsp", "SyncError")


class SyncError(*((_KK_SYNC_ERROR,) if _KK_SYNC_ERROR else (RuntimeError,))):
    """Raised when the receiver cannot align to the reference sequence
    (kkmodem.rxdsp.SyncError, rxdsp.py:63; a subclass of it when kkmodem is
    importable)."""


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int
_F = ctypes.c_float
_D = ctypes.c_double
_SZ = ctypes.c_size_t
_U64 = ctypes.c_uint64

_SIGS = {
    "kk_last_error": ([], ctypes.c_char_p),
    "kk_version": ([], _I),
    "kk_device_sync": ([], _I),
    "kk_launch_count": ([], ctypes.c_ulonglong),
    "kk_fma_peak": ([_P, _P], _I),
    "kk_upload": ([_P, _P, _I64, _P], _I),
    "kk_reconstruct_pairs": ([_I, _P, _F, _F, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _I, _I, _P, _U64, _I,
                              _P], _I),
    "kk_unpack12": ([_P, _I64, _P, _P], _I),
    "kk_frequency_shift": ([_P, _P, _I64, _D, _D, _I64, _P], _I),
    "kk_carrier_means": ([_P, _I64, _I, _I64, _I64, _I, _P, _P], _I),
    "kk_static_blocks": ([_P, _I64, _I64, _I64, _I64, _P, _I64, _I, _I, _I, _I, _P, _U64, _I, _P, _P, _P, _P], _I),
    "kk_symbol_sync_scratch_bytes": ([_I64, _I], _SZ),
    "kk_symbol_sync": ([_P, _I64, _P, _I, _I64, _P, _P, _SZ, _P], _I),
    "kk_symbol_sync_enqueue": ([_P, _I64, _P, _I, _I64, _P, _P, _SZ, _P], _I),
    "kk_ddlms_sequential": ([_P, _I64, _F, _I, _P, _I64, _P, _P, _I, _P, _P, _I, _F, _F, _F, _I, _F, _I,
                             _P, _P, _P, _P], _I),
    "kk_ddlms_workspace_bytes": ([_I64, _I], _SZ),
    "kk_ddlms_solve": ([_P, _I64, _F, _P, _I64, _P, _I, _P, _P, _I, _F, _F, _F, _I, _F, _I, _I, _F, _P, _P,
                        _P, _P, _SZ, _P, _P], _I),
    "kk_ddlms_solve_async": ([_P, _I64, _F, _P, _I64, _P, _P, _I, _P, _P, _I, _F, _F, _F, _I, _F, _I, _I, _I,
                              _F, _P, _P, _P, _SZ, _P, _P], _I),
    "kk_ddlms_create": ([_P, _I64, _F, _P, _I64, _I, _P, _P, _I, _F, _F, _F, _F, _I, _F, _P, _SZ, _P], _P),
    "kk_ddlms_train": ([_P, _P, _P], _I),
    "kk_ddlms_speculate": ([_P, _P, _P], _I),
    "kk_ddlms_iterate": ([_P, _P, _I, _P, _P, _P], _I),
    "kk_ddlms_bind_outputs": ([_P, _P, _P], _I),
    "kk_ddlms_finish": ([_P, _P, _P, _P, _P], _I),
    "kk_ddlms_destroy": ([_P], None),
    "kk_bit_errors": ([_P, _P, _I64, _P, _I64, _P, _P, _I64, _I64, _I64, _P, _P], _I),
    "kk_demap": ([_P, _I64, _I, _P, _P, _P, _P], _I),
    "kk_pack_bits": ([_P, _I64, _I64, _P, _I64, _I, _P, _I, _P, _P], _I),
    "kk_bit_xcorr_workspace_bytes": ([_I64, _I64, _I], _SZ),
    "kk_bit_xcorr": ([_P, _I64, _P, _I64, _I, _P, _SZ, _P, _P], _I),
    "kk_label_bits": ([_P, _I64, _P, _I, _I, _P, _P], _I),
    "kk_bit_error_windows": ([_P, _P, _I64, _I64, _P, _P, _P], _I),
    "kk_evm_sums": ([_P, _P, _I64, _P, _P, _P], _I),
    "kk_fft_workspace_bytes": ([_I64, _I64], _SZ),
    "kk_fft": ([_P, _P, _I64, _I64, _I, _P, _SZ, _P], _I),
    "kk_ssfm_workspace_bytes": ([_I64], _SZ),
    "kk_ssfm_span": ([_P, _I64, ctypes.c_double, _I, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                      ctypes.c_double, _P, _SZ, _P], _I),
}

class K1Job(ctypes.Structure):
    """kk_k1_job (include/kkb200.h): one stream's kk_reconstruct_pairs arguments."""
    _fields_ = [("in_", _P), ("in_scale", _F), ("clamp_rel", _F), ("n_hops", _I64), ("st_u", _P), ("st_a", _P),
                ("st_dead", _P), ("new_u", _P), ("new_a", _P), ("new_dead", _P), ("out", _P), ("hop_sum", _P),
                ("hop_dead", _P), ("clamped", _P), ("n0_global", _I64), ("rot_p", _I), ("rot_q", _I),
                ("rot_tab", _P), ("rot_step", _U64), ("mirror", _I)]


class K2Job(ctypes.Structure):
    """kk_k2_job (include/kkb200.h): one stream's kk_static_blocks arguments."""
    _fields_ = [("z", _P), ("z_index0", _I64), ("hb0", _I64), ("n_blocks", _I64), ("valid_end", _I64),
                ("seg_mean", _P), ("seg_index0", _I64), ("seg_len", _I), ("carrier", _I), ("rot_p", _I),
                ("rot_q", _I), ("rot_tab", _P), ("rot_step", _U64), ("mirror", _I), ("h_even", _P), ("h_odd", _P),
                ("out", _P)]


_SIGS["kk_reconstruct_pairs_batch"] = ([_I, ctypes.POINTER(K1Job), _I, _P], _I)
_SIGS["kk_static_blocks_batch"] = ([ctypes.POINTER(K2Job), _I, _P], _I)

EXPORTED = sorted(_SIGS)
_lib = None


def load():
    """Load (once) and return the ctypes library; raises if unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("KKB200_LIB") or LIB_PATH   # variant builds (tools/) only
    if not os.path.exists(path):
        raise RuntimeError(
            f"CUDA library {path} is missing: build it with "
            "`python -m paper_2108_07001_b200.build` (no CPU fallback exists)")
    lib = ctypes.CDLL(path)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def check(rc: int, what: str = "") -> None:
    if rc == KK_OK:
        return
    msg = load().kk_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == KK_ERR_PARAM:
        raise ParameterError(text)
    if rc == KK_ERR_SYNC:
        raise SyncError(text)
    raise RuntimeError(text)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)
