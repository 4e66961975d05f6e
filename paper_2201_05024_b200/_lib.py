"""ctypes binding of the C ABI in ``include/kapsm_b200.h``.

The library ``paper_2201_05024_b200/lib/libkapsm_b200.so`` is built in-tree by
``paper_2201_05024_b200/build.py`` (sm_100a).  There is no fallback: if the
library is missing or CUDA is unavailable, every compute call raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libkapsm_b200.so")

KAPSM_OK = 0
KAPSM_ERR_INVALID = 1
KAPSM_ERR_CUDA = 2
KAPSM_ERR_UNSUPPORTED = 3
TRAIN_DEGENERATE = 1
TRAIN_STALLED = 2


class KernelParamsC(C.Structure):
    _fields_ = [("w_l", C.c_double), ("w_g", C.c_double), ("sigma_sq", C.c_double)]


_P = C.c_void_p
_I = C.c_int
_LL = C.c_longlong
_D = C.c_double
_KP = KernelParamsC

# name -> (restype, argtypes); one entry per symbol of include/kapsm_b200.h
SIGNATURES = {
    "kapsm_strerror": (C.c_char_p, [_I]),
    "kapsm_abi_version": (_I, []),
    "kapsm_max_window": (_I, []),
    "kapsm_max_samples": (_I, []),
    "kapsm_pilot_gram_f32": (_I, [_P, _LL, _I, _I, _I, _KP, _P, _LL, _LL, _P]),
    "kapsm_pilot_gram_f64": (_I, [_P, _LL, _I, _I, _I, _KP, _P, _LL, _LL, _P]),
    "kapsm_sample_gram_f32": (_I, [_P, _LL, _I, _I, _I, _KP, _P, _LL, _LL, _P]),
    "kapsm_sample_gram_f64": (_I, [_P, _LL, _I, _I, _I, _KP, _P, _LL, _LL, _P]),
    "kapsm_train_f32": (_I, [_P, _LL, _LL, _P, _LL, _P, _LL, _I, _P, _I, _I, _I, _I, _D, _KP,
                             _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "kapsm_train_f64": (_I, [_P, _LL, _LL, _P, _LL, _P, _LL, _I, _P, _I, _I, _I, _I, _D, _KP,
                             _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "kapsm_train_general_f32": (_I, [_P, _LL, _LL, _P, _LL, _P, _LL, _I, _P, _I, _I, _I, _I, _D,
                                     _KP, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "kapsm_train_general_f64": (_I, [_P, _LL, _LL, _P, _LL, _P, _LL, _I, _P, _I, _I, _I, _I, _D,
                                     _KP, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "kapsm_detect_frames_f32": (_I, [_P, _LL, _I, _I, _I, _I, _I, _P, _P, _KP, _P, _I, _I, _P,
                                     _P, _P, _P, _P, _P]),
    "kapsm_detect_frames_f64": (_I, [_P, _LL, _I, _I, _I, _I, _I, _P, _P, _KP, _P, _I, _I, _P,
                                     _P, _P, _P, _P, _P]),
    "kapsm_run_frames_f32": (_I, [_P, _LL, _P, _P, _I, _I, _I, _I, _I, _I, _D, _KP, _P, _P, _I,
                                  _I, _P, _LL, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "kapsm_run_frames_f64": (_I, [_P, _LL, _P, _P, _I, _I, _I, _I, _I, _I, _D, _KP, _P, _P, _I,
                                  _I, _P, _LL, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "kapsm_screen_workspace_bytes": (_LL, [_I, _I, _I]),
    "kapsm_pipeline_workspace_bytes": (_LL, [_I, _I, _I, _I, _I, _I]),
    "kapsm_stream_create": (_I, [C.POINTER(C.c_void_p)]),
    "kapsm_stream_destroy": (_I, [_P]),
    "kapsm_stream_frame_in": (_I, [_P, _P, _P, _P, _P, _P, _I, _P, _P, _P, _P, _P, _P, _P]),
    "kapsm_stream_frame_out": (_I, [_P, _P, _I, _P, _P, _P, _P]),
    "kapsm_detect_screen_f32": (_I, [_P, _LL, _I, _I, _I, _I, _KP, _P, _P]),
    "kapsm_detect_screen_f64": (_I, [_P, _LL, _I, _I, _I, _I, _KP, _P, _P]),
    "kapsm_detect_finish_f32": (_I, [_P, _LL, _I, _I, _I, _I, _I, _P, _P, _KP, _P, _I, _I, _P,
                                     _P, _P, _P, _P, _P, _P]),
    "kapsm_detect_finish_f64": (_I, [_P, _LL, _I, _I, _I, _I, _I, _P, _P, _KP, _P, _I, _I, _P,
                                     _P, _P, _P, _P, _P, _P]),
    "kapsm_run_frames_overlap_f32": (_I, [_P, _LL, _P, _P, _I, _I, _I, _I, _I, _I, _D, _KP, _P,
                                          _P, _I, _I, _P, _LL, _P, _P, _P, _P, _P, _P, _P, _P,
                                          _P, _P, _P, _P]),
    "kapsm_run_frames_overlap_f64": (_I, [_P, _LL, _P, _P, _I, _I, _I, _I, _I, _I, _D, _KP, _P,
                                          _P, _I, _I, _P, _LL, _P, _P, _P, _P, _P, _P, _P, _P,
                                          _P, _P, _P, _P]),
    "kapsm_batch_evaluate_f32": (_I, [_P, _P, _P, _I, _I, _P, _I, _KP, _P, _P]),
    "kapsm_batch_evaluate_f64": (_I, [_P, _P, _P, _I, _I, _P, _I, _KP, _P, _P]),
    "kapsm_batch_detect_f32": (_I, [_P, _P, _P, _I, _I, _P, _I, _KP, _P, _P]),
    "kapsm_batch_detect_f64": (_I, [_P, _P, _P, _I, _I, _P, _I, _KP, _P, _P]),
    "kapsm_demap_f32": (_I, [_P, _LL, _P, _I, _P, _P]),
    "kapsm_demap_f64": (_I, [_P, _LL, _P, _I, _P, _P]),
    "kapsm_count_mismatch": (_I, [_P, _P, _LL, _I, _P, _P]),
    "kapsm_targets_from_labels_f32": (_I, [_P, _LL, _P, _I, _P, _P]),
    "kapsm_targets_from_labels_f64": (_I, [_P, _LL, _P, _I, _P, _P]),
    # internal instrumentation (not in the public header)
    "kapsm_internal_fp32_peak": (_I, [_P, _I, _I, _P]),
    "kapsm_internal_run_frames_overlap_mode_f32": (_I, [_I, _P, _LL, _P, _P, _I, _I, _I, _I, _I,
                                                        _I, _D, _KP, _P, _P, _I, _I, _P, _LL, _P,
                                                        _P, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                                                        _P]),
    "kapsm_internal_train_tp_ws_bytes": (_LL, [_I, _I, _I]),
    "kapsm_internal_train_tp_f32": (_I, [_I, _P, _LL, _P, _I, _I, _I, _I, _I, _D, _KP, _P, _P, _P,
                                         _P, _P, _P, _P, _P]),
    "kapsm_internal_screen_simt_f32": (_I, [_P, _LL, _I, _I, _I, _I, _KP, _P, _P]),
}

_lib = None
_lock = threading.Lock()


def load():
    """Load (once) and return the ctypes handle; raises if the library is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"kapsm CUDA library not built ({LIB_PATH}); run "
                "`python -m paper_2201_05024_b200.build` (there is no CPU fallback)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(code: int, what: str):
    if code != KAPSM_OK:
        msg = load().kapsm_strerror(code).decode()
        if code == KAPSM_ERR_INVALID:
            raise ValueError(f"{what}: {msg}")
        if code == KAPSM_ERR_UNSUPPORTED:
            raise NotImplementedError(f"{what}: {msg}")
        raise RuntimeError(f"{what}: {msg}")


def params(p) -> KernelParamsC:
    return KernelParamsC(float(p.w_l), float(p.w_g), float(p.sigma_sq))
