"""ctypes binding of libmshbm.so (the C ABI in include/mshbm.h).

The product path has no CPU fallback: if the shared library cannot be loaded
or no CUDA device is visible, every entry point raises RuntimeError.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmshbm.so")

MSHBM_OK = 0
MSHBM_ERR_VALUE = 1
MSHBM_ERR_CONFIG = 2
ABI_VERSION = 2        # include/mshbm.h MSHBM_ABI_VERSION
IO_DEVICE = 0
IO_HOST = 1
FLAG_TIMING = 1
FLAG_NO_GRAPH = 2


MSHBM_ERR_DECODE = 10
MSHBM_ERR_MALFORMED = 11
MSHBM_ERR_TRUNCATED = 12
MSHBM_ERR_MAXVAL = 13
MSHBM_ERR_MISSING_KEY = 14


class PnmHeader(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("maxval", C.c_int32),
                ("channels", C.c_int32), ("ascii", C.c_int32), ("itemsize", C.c_int32),
                ("payload_offset", C.c_int64)]


class PfmHeader(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("scale", C.c_double),
                ("payload_offset", C.c_int64)]


class Config(C.Structure):
    _fields_ = [("d_max", C.c_int32), ("levels", C.c_int32), ("block", C.c_int32),
                ("radius", C.c_int32), ("alpha", C.c_double), ("beta", C.c_double),
                ("sigma_eps", C.c_double), ("sign", C.c_int32), ("reserved", C.c_int32)]


class LevelTraceC(C.Structure):
    _fields_ = [("level", C.c_int32), ("height", C.c_int32), ("width", C.c_int32),
                ("d_max", C.c_int32), ("block", C.c_int32), ("reserved", C.c_int32),
                ("trusted", C.c_int64), ("trusted_evals", C.c_int64),
                ("trusted_window_max", C.c_int64), ("full_search_pixels", C.c_int64),
                ("selection_evals", C.c_int64), ("refined", C.c_int64),
                ("refine_evals", C.c_int64), ("median_replaced", C.c_int64),
                ("ms_upsample", C.c_float), ("ms_select", C.c_float),
                ("ms_refine", C.c_float), ("ms_median", C.c_float),
                ("ms_build", C.c_float), ("ms_total", C.c_float)]


P = C.c_void_p
I32 = C.c_int32
I64 = C.c_int64
D = C.c_double

# name -> (restype, argtypes); every symbol include/mshbm.h declares
SIGNATURES = {
    "mshbm_abi_version": (C.c_int, []),
    "mshbm_status_string": (C.c_char_p, [C.c_int]),
    "mshbm_last_error": (C.c_char_p, [P]),
    "mshbm_create": (C.c_int, [C.POINTER(P), C.c_int]),
    "mshbm_destroy": (C.c_int, [P]),
    "mshbm_launch_count": (I64, [P]),
    "mshbm_level_d_max": (I32, [I32, I32]),
    "mshbm_level_block": (I32, [I32, I32]),
    "mshbm_auto_levels": (C.c_int, [I64, I64, I64, I64, C.POINTER(I32)]),
    "mshbm_resolve_levels": (C.c_int, [C.POINTER(Config), I32, I32, C.POINTER(I32)]),
    "mshbm_downsample": (C.c_int, [P, P, I32, I32, I64, P, I64, P]),
    "mshbm_binomial_smooth": (C.c_int, [P, P, I32, I32, I64, P, I64, P]),
    "mshbm_run_pipeline": (C.c_int, [P, P, P, I32, I32, I64, C.POINTER(Config), P, P, I64,
                                     P, C.POINTER(I32), I32, I32, P]),
    "mshbm_run_pipeline_band": (C.c_int, [P, P, P, I32, I32, I64, C.POINTER(Config), I32, I32, P,
                                          P, I64, P, C.POINTER(I32), I32, I32, P]),
    "mshbm_run_batch": (C.c_int, [P, I32, P, P, I32, I32, I64, C.POINTER(Config), P, P, I64, P,
                                  I32, I32, P]),
    "mshbm_run_pyramid": (C.c_int, [P, I32, P, P, P, P, P, P, P, C.POINTER(Config), P, P,
                                    I64, P, P]),
    "mshbm_engine_create": (C.c_int, [P, P, P, I32, I32, I64, I32, I32, D, I32, C.POINTER(P)]),
    "mshbm_engine_destroy": (C.c_int, [P]),
    "mshbm_engine_stats": (C.c_int, [P, P, P, P, P, P]),
    "mshbm_engine_plane": (C.c_int, [P, I32, P, P]),
    "mshbm_engine_at": (C.c_int, [P, P, P, P, I64, P, P]),
    "mshbm_engine_dsi_rows": (C.c_int, [P, P, P, I64, P, P]),
    "mshbm_match_coarsest": (C.c_int, [P, P, P, P]),
    "mshbm_select_with_prior": (C.c_int, [P, P, P, D, I32, P, P, P, P]),
    "mshbm_refine_level": (C.c_int, [P, P, P, D, P, P, P, P]),
    "mshbm_selective_median": (C.c_int, [P, P, P, I32, I32, D, P, P, P]),
    "mshbm_upsample_prior": (C.c_int, [P, P, P, I32, I32, I32, I32, P, P, P]),
    "mshbm_pnm_parse": (C.c_int, [P, I64, C.POINTER(PnmHeader)]),
    "mshbm_pnm_decode": (C.c_int, [P, I64, C.POINTER(PnmHeader), P, I64]),
    "mshbm_pnm_upload": (C.c_int, [P, I64, C.POINTER(PnmHeader), P, I64, P]),
    "mshbm_pfm_parse": (C.c_int, [P, I64, C.POINTER(PfmHeader)]),
    "mshbm_pfm_decode": (C.c_int, [P, I64, C.POINTER(PfmHeader), P, P, I64]),
    "mshbm_pfm_encode": (I64, [P, I32, I32, I64, D, P, I64]),
    "mshbm_pgm_encode": (I64, [P, I32, I32, I64, I32, D, P, I64]),
    "mshbm_evaluate": (C.c_int, [P, P, P, P, I64, D, C.POINTER(D), C.POINTER(I64), C.POINTER(D),
                                 P]),
    "mshbm_probe_fp32_peak": (C.c_int, [C.c_int, C.c_int, C.POINTER(D), C.POINTER(D)]),
    "mshbm_probe_fp64_peak": (C.c_int, [C.c_int, C.c_int, C.POINTER(D), C.POINTER(D)]),
}

_lock = threading.Lock()
_lib = None
_ctx = {}


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Load libmshbm.so and bind every ABI symbol (no device needed)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise RuntimeError(
                f"libmshbm.so not found at {path}: build it with "
                "`python -m paper_1901_09593_b200.build` (there is no CPU fallback)")
        lib = C.CDLL(path)
        lib.mshbm_abi_version.restype = C.c_int
        if lib.mshbm_abi_version() != ABI_VERSION:
            raise RuntimeError(f"{path} has ABI {lib.mshbm_abi_version()}, this binding expects "
                               f"{ABI_VERSION}: rebuild with `python -m paper_1901_09593_b200.build`")
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def lib() -> C.CDLL:
    return _lib if _lib is not None else load_library()


class MshbmError(RuntimeError):
    pass


def check(status: int, ctx=None) -> None:
    """Map an mshbm_status to the reference's exception types."""
    if status == MSHBM_OK:
        return
    msg = lib().mshbm_last_error(ctx)
    msg = msg.decode() if msg else lib().mshbm_status_string(status).decode()
    if status == MSHBM_ERR_CONFIG:
        from .matcher import ConfigError
        raise ConfigError(msg)
    if status == MSHBM_ERR_VALUE:
        raise ValueError(msg)
    raise MshbmError(f"libmshbm: {msg}")


def context(device: int | None = None):
    """Process-wide mshbm context for ``device`` (default: current CUDA device)."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1901_09593_b200 needs a CUDA device (B200); none is visible "
                           "and there is no CPU fallback")
    if device is None:
        device = torch.cuda.current_device()
    with _lock:
        ctx = _ctx.get(device)
    if ctx is not None:
        return ctx
    h = P()
    check(lib().mshbm_create(C.byref(h), int(device)))
    with _lock:
        _ctx[device] = h
    return h


def launch_count(device: int | None = None) -> int:
    return int(lib().mshbm_launch_count(context(device)))


def current_stream():
    import torch
    return P(torch.cuda.current_stream().cuda_stream)
