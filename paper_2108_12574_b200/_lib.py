"""ctypes binding of the C-ABI in include/iedd_b200.h.

The library is built in-tree (paper_2108_12574_b200/build.py).  There is no
CPU fallback: if the .so is missing or no CUDA device is visible, the calls
that need the device raise."""

from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IEDD_B200_LIB") or os.path.join(HERE, "libiedd_b200.so")  # override: A/B builds

IE_OK = 0
IE_ERR_ARG = -1
IE_ERR_NOT_SPD = 1
IE_ERR_BREAKDOWN = 2
IE_ERR_NONFINITE = 3
IE_ERR_NO_RITZ = 4
IE_ERR_CUDA = 5

VARIANTS = {"packed_inverse": 0, "subst": 1}
MATVEC_METHODS = {"direct": 0, "fft": 1}


class IeGeom(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("n", ctypes.c_int32), ("spacing", ctypes.c_double),
                ("weight", ctypes.c_double), ("diag", ctypes.c_double)]


_lib = None

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_D = ctypes.c_double

_SIGS = {
    "ie_matvec_create": (_I32, [ctypes.POINTER(IeGeom), ctypes.POINTER(_P)]),
    "ie_matvec_create_method": (_I32, [ctypes.POINTER(IeGeom), _I32, ctypes.POINTER(_P)]),
    "ie_matvec_destroy": (None, [_P]),
    "ie_matvec_f64": (_I32, [_P, _P, _I64, _I32, _P, _I64, _I64, _I64, _P]),
    "ie_matvec_band_fwd_f64": (_I32, [_P, _P, _I64, _I32, _I64, _I64, _I32, _P, _P, _P]),
    "ie_matvec_band_cols_f64": (_I32, [_P, _P, _I64, _I64, _P]),
    "ie_matvec_band_inv_f64": (_I32, [_P, _P, _I64, _I64, _I32, _P, _I64, _I32, _P, _P]),
    "ie_absmax_partials_f64": (_I32, [_P, _I64, _I64, _P, _P]),
    "ie_shard_create": (_I32, [_P, _P, _I32, _I32, _P, _P, ctypes.POINTER(_P)]),
    "ie_shard_destroy": (None, [_P]),
    "ie_shard_need_rows": (_I32, [_P, _P]),
    "ie_shard_handle_bytes": (_I64, []),
    "ie_shard_export": (_I32, [_P, _P]),
    "ie_shard_connect": (_I32, [_P, _P]),
    "ie_shard_connect_local": (_I32, [_P, _I32]),
    "ie_pcg_sharded_f64": (_I32, [_P, _P, _P, _D, _I64, _P, ctypes.POINTER(_I64), _P, _P,
                                  ctypes.POINTER(_I64), ctypes.POINTER(_D), _P]),
    "ie_pcg_sharded_local_f64": (_I32, [_P, _I32, _P, _P, _D, _I64, _P, ctypes.POINTER(_I64), _P, _P,
                                        ctypes.POINTER(_I64), ctypes.POINTER(_D), _P]),
    "ie_assemble_block_f64": (_I32, [ctypes.POINTER(IeGeom), _P, _I64, _P, _I64, _P, _P]),
    "ie_precond_create": (_I32, [ctypes.POINTER(IeGeom), _P, _P, _I64, _I32, _I32, ctypes.POINTER(_P),
                                 ctypes.POINTER(_I64), _P]),
    "ie_precond_destroy": (None, [_P]),
    "ie_precond_apply_f64": (_I32, [_P, _P, _P, _P]),
    "ie_precond_stats": (_I32, [_P, _P]),
    "ie_precond_block_f64": (_I32, [_P, _I64, _P, ctypes.POINTER(_I64), ctypes.POINTER(_I32)]),
    "ie_pcg_f64": (_I32, [_P, _P, _P, _P, _D, _I64, _P, ctypes.POINTER(_I64), _P, _P,
                          ctypes.POINTER(_I64), ctypes.POINTER(_D), _P]),
    "ie_pcg_host_f64": (_I32, [_P, _P, _P, _P, _D, _I64, _P, ctypes.POINTER(_I64), _P, _P,
                          ctypes.POINTER(_I64), ctypes.POINTER(_D), _P]),
    "ie_pcg_profile_f64": (_I32, [_P, _P, _P, _P, _D, _I64, _P, ctypes.POINTER(_I64), _P, _P, _P, _P]),
    "ie_lanczos_f64": (_I32, [_P, _P, _P, _I32, _I64, _D, ctypes.POINTER(_D), ctypes.POINTER(_I64), _P]),
    "ie_fp64_peak": (_I32, [ctypes.POINTER(_D), _P]),
    "ie_dmma_peak": (_I32, [ctypes.POINTER(_D), _P]),
    "ie_dot_chunk": (_I64, []),
    "ie_dot_partials_f64": (_I32, [_P, _P, _I64, _I32, _P, _P]),
    "ie_sum_partials_f64": (_I32, [_P, _I64, _P, _P]),
    "ie_update_f64": (_I32, [_I32, _P, _P, _D, _I64, _P]),
    "ie_line_partials_f64": (_I32, [_P, _P, _I64, _I32, _I32, _I32, _P, _P]),
    "ie_last_error": (ctypes.c_char_p, []),
    "ie_launch_count": (_I64, []),
}


def lib():
    """Load libiedd_b200.so (raises ImportError if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the sm_100a extension first "
                "(python -c 'import __graft_entry__ as g; g.build()')")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    return lib().ie_last_error().decode(errors="replace")


def launch_count() -> int:
    return int(lib().ie_launch_count())


def check(rc: int, what: str):
    if rc == IE_OK:
        return
    msg = last_error()
    if rc < 0:
        raise ValueError(f"{what}: {msg}")
    raise RuntimeError(f"{what} failed (code {rc}): {msg}")


def torch_cuda():
    """The torch module with a usable CUDA device (raises otherwise)."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2108_12574_b200 needs a CUDA device (B200, sm_100a); none is visible")
    return torch


def stream_ptr():
    torch = torch_cuda()
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def np_ptr(a: np.ndarray) -> ctypes.c_void_p:
    return a.ctypes.data_as(ctypes.c_void_p)
