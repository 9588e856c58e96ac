"""ctypes binding of the C-ABI (include/monoalign_b200.h).

The in-tree ``_lib/libmonoalign_b200.so`` is the only implementation: if it
is missing or cannot be loaded this module raises -- there is no CPU
fallback.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MAS_LIB_PATH") or os.path.join(_HERE, "_lib", "libmonoalign_b200.so")

MAS_OK = 0
MAS_E_VALIDATION = 1
MAS_E_IO = 2
MAS_E_CUDA = 3
MAS_E_UNSUPPORTED = 4

MAS_ENGINE_REFERENCE = 0
MAS_ENGINE_PARALLEL = 1
MAS_FLAG_UNCHECKED = 0x1
MAS_FLAG_NO_CHECK = 0x2
MAS_FLAG_PIPELINED = 0x4
MAS_PART_FORWARD = 0x1
MAS_PART_BACKTRACK = 0x2
MAS_PART_ALL = 0x3
MAS_IO_DEFAULT_BYTE_BUDGET = 1 << 30

# include/monoalign/errors.hpp:8-30 of the reference, declaration order.
ERRC_NAMES = (
    "ZeroDim", "InfeasibleLengths", "LengthsOutOfRange", "NonFinite", "SpeechTooLong",
    "ShapeMismatch", "InvalidPath", "InvalidMatrix", "InvalidConfig", "TooLarge",
    "EmptyReport", "InsufficientPoints", "IoFailure", "BadMagic", "UnsupportedVersion",
    "TruncatedFile", "DimensionOverflow",
)


class MasError(ctypes.Structure):
    _fields_ = [
        ("status", ctypes.c_int32),
        ("errc", ctypes.c_int32),
        ("item", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("i", ctypes.c_int64),
        ("j", ctypes.c_int64),
        ("message", ctypes.c_char * 512),
    ]


class MasConfig(ctypes.Structure):
    _fields_ = [
        ("engine", ctypes.c_int32),
        ("max_neg_val", ctypes.c_float),
        ("lane_padding", ctypes.c_int32),
        ("threads", ctypes.c_int32),
        ("flags", ctypes.c_uint32),
    ]


# Every symbol include/monoalign_b200.h declares, with its ctypes signature.
_VP = ctypes.c_void_p
_SIGS = {
    "mas_config_default": (None, [ctypes.POINTER(MasConfig)]),
    "mas_align_host": (ctypes.c_int, [_VP, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _VP,
                                      ctypes.POINTER(MasConfig), _VP, _VP,
                                      ctypes.POINTER(MasError)]),
    "mas_align_host_ex": (ctypes.c_int, [_VP, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                         _VP, ctypes.POINTER(MasConfig), _VP, _VP, _VP,
                                         ctypes.POINTER(MasError)]),
    "mas_align_device": (ctypes.c_int, [_VP, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                        ctypes.c_int32, _VP, ctypes.POINTER(MasConfig), _VP, _VP,
                                        _VP, ctypes.POINTER(MasError)]),
    "mas_align_device_ex": (ctypes.c_int, [_VP, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                           ctypes.c_int32, _VP, ctypes.POINTER(MasConfig), _VP,
                                           _VP, _VP, _VP, ctypes.POINTER(MasError)]),
    "mas_plan_create": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                       ctypes.c_int64, _VP, ctypes.POINTER(MasConfig),
                                       ctypes.POINTER(_VP), ctypes.POINTER(MasError)]),
    "mas_plan_enqueue": (ctypes.c_int, [_VP, _VP, _VP, _VP, _VP, ctypes.POINTER(MasError)]),
    "mas_plan_enqueue_part": (ctypes.c_int, [_VP, ctypes.c_uint32, _VP, _VP, _VP, _VP,
                                             ctypes.POINTER(MasError)]),
    "mas_plan_enqueue_ex": (ctypes.c_int, [_VP, ctypes.c_uint32, _VP, _VP, _VP, _VP, _VP,
                                           ctypes.POINTER(MasError)]),
    "mas_plan_finish": (ctypes.c_int, [_VP, _VP, _VP, ctypes.POINTER(MasError)]),
    "mas_plan_launches": (ctypes.c_int, [_VP]),
    "mas_plan_geometry": (None, [_VP, ctypes.POINTER(ctypes.c_int32 * 6)]),
    "mas_plan_destroy": (None, [_VP]),
    "mas_generate_device": (ctypes.c_int, [ctypes.c_uint64, ctypes.c_int32, ctypes.c_int32,
                                           ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, _VP,
                                           _VP]),
    "mas_validate_config": (ctypes.c_int, [ctypes.POINTER(MasConfig), ctypes.POINTER(MasError)]),
    "mas_validate_host": (ctypes.c_int, [_VP, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _VP,
                                         ctypes.c_int32, ctypes.POINTER(MasError)]),
    "mas_io_read_header": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_uint64,
                                          ctypes.POINTER(ctypes.c_int32),
                                          ctypes.POINTER(ctypes.c_int64 * 3),
                                          ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(MasError)]),
    "mas_io_read": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_int32,
                                   ctypes.POINTER(ctypes.c_int64 * 3), _VP, _VP,
                                   ctypes.POINTER(MasError)]),
    "mas_io_write": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int32, ctypes.c_int64,
                                    ctypes.c_int64, ctypes.c_int64, _VP, _VP,
                                    ctypes.POINTER(MasError)]),
    "mas_forward_scores": (ctypes.c_int, [_VP, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                          ctypes.c_int32, _VP, ctypes.c_float, _VP,
                                          ctypes.POINTER(MasError)]),
    "mas_forward_scores_ex": (ctypes.c_int, [_VP, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                             ctypes.c_int32, _VP, ctypes.c_int32, ctypes.c_float,
                                             _VP, ctypes.POINTER(MasError)]),
    "mas_backtrack_scores": (ctypes.c_int, [_VP, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                            ctypes.c_int32, _VP, _VP, _VP,
                                            ctypes.POINTER(MasError)]),
    "mas_relax_column": (ctypes.c_int, [_VP, _VP, ctypes.c_int32, ctypes.c_float, _VP,
                                        ctypes.POINTER(MasError)]),
    "mas_gaussian_loglik_device": (ctypes.c_int, [_VP, _VP, _VP, ctypes.c_int32, ctypes.c_int32,
                                                  ctypes.c_int32, ctypes.c_int32, _VP,
                                                  ctypes.c_int64, _VP, ctypes.POINTER(MasError)]),
    "mas_align_gaussian_device": (ctypes.c_int, [_VP, _VP, _VP, ctypes.c_int32, ctypes.c_int32,
                                                 ctypes.c_int32, ctypes.c_int32, _VP,
                                                 ctypes.POINTER(MasConfig), _VP, _VP, _VP, _VP,
                                                 ctypes.POINTER(MasError)]),
    "mas_plan_create_gaussian": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                                ctypes.c_int32, _VP, ctypes.POINTER(MasConfig),
                                                ctypes.POINTER(ctypes.c_void_p),
                                                ctypes.POINTER(MasError)]),
    "mas_plan_enqueue_gaussian": (ctypes.c_int, [_VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP,
                                                 ctypes.POINTER(MasError)]),
    "mas_errc_name": (ctypes.c_char_p, [ctypes.c_int32]),
    "mas_abi_version": (ctypes.c_int, []),
}

_lib = None


def load() -> ctypes.CDLL:
    """Loads the in-tree library (building it first if it is absent and nvcc
    is available).  Raises if the CUDA library cannot be provided."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        from . import build as _build
        _build.build()
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def raise_for(rc: int, err: MasError) -> None:
    if rc == MAS_OK:
        return
    msg = err.message.decode(errors="replace")
    if rc == MAS_E_VALIDATION:
        raise ValueError(msg)
    if rc == MAS_E_IO:
        raise OSError(msg)
    raise RuntimeError(f"monoalign device path failed (status {rc}): {msg}")
