"""ctypes binding of the C ABI (include/tmatch_cuda.h) -- libtmatch_cuda.so.

There is no fallback: if the in-tree library is missing, importing the product API raises;
if no sm_100a device is present, creating a context raises NoDeviceError.
"""
from __future__ import annotations

import ctypes as C
import os
import re

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB_PATH = os.path.join(PKG, "lib", "libtmatch_cuda.so")
API_LIB_PATH = os.path.join(PKG, "lib", "libtmatch.so")
HEADER = os.path.join(ROOT, "include", "tmatch_cuda.h")

TM_OK, TM_EINVAL, TM_ECUDA, TM_ENODEV, TM_ENOMEM = 0, -1, -2, -3, -4
MODE = {"brute": 0, "egs": 1, "opta": 2}
POLICY = {"reference": 0, "frozen": 1, "sequential": 2, "seeded": 3}
TM_MAX_TRACE = 64


class TmatchError(RuntimeError):
    pass


class InvalidArgument(TmatchError, ValueError):
    """The reference's std::invalid_argument (same message text)."""


class NoDeviceError(TmatchError):
    pass


class MatchResult(C.Structure):
    _fields_ = [("mode", C.c_int32), ("best_row", C.c_int32), ("best_col", C.c_int32),
                ("best_degenerate", C.c_int32), ("best_rho", C.c_double),
                ("refined_row", C.c_int32), ("refined_col", C.c_int32),
                ("refined_rho", C.c_double), ("below_threshold", C.c_int32),
                ("extent_rows", C.c_int32), ("extent_cols", C.c_int32), ("_pad0", C.c_int32),
                ("final_threshold", C.c_double), ("centers", C.c_int64),
                ("eliminated", C.c_int64), ("retained", C.c_int64), ("ops", C.c_int64),
                ("elim_pct", C.c_double), ("wall_ms", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if not k.startswith("_")}

    def __repr__(self):
        d = self.as_dict()
        return "MatchResult(" + ", ".join(f"{k}={v}" for k, v in d.items()) + ")"


class MatchParams(C.Structure):
    _fields_ = [("mode", C.c_int32), ("h0", C.c_int32), ("w0", C.c_int32),
                ("has_init_threshold", C.c_int32), ("init_threshold", C.c_double),
                ("rho_th", C.c_double), ("rho_max", C.c_double), ("xi_fraction", C.c_double),
                ("opta_margin", C.c_double), ("kernel_profile", C.POINTER(C.c_double)),
                ("kernel_len", C.c_int32), ("parallel", C.c_int32), ("threads", C.c_int32),
                ("record_visits", C.c_int32), ("policy", C.c_int32), ("max_group", C.c_int32),
                ("seed_margin", C.c_double)]


class EgsIter(C.Structure):
    _fields_ = [("h", C.c_int32), ("w", C.c_int32), ("central", C.c_double),
                ("retained", C.c_int64), ("retained_cost", C.c_double),
                ("amortized", C.c_double), ("total", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class OptaIter(C.Structure):
    _fields_ = [("h", C.c_int32), ("w", C.c_int32), ("cost", C.c_double),
                ("restored", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class PrepInfo(C.Structure):
    _fields_ = [("mode", C.c_int32), ("m", C.c_int32), ("n", C.c_int32), ("h", C.c_int32),
                ("w", C.c_int32), ("extent_rows", C.c_int32), ("extent_cols", C.c_int32),
                ("kappa", C.c_int32), ("lambda_", C.c_double), ("cost", EgsIter),
                ("egs_trace_len", C.c_int32), ("egs_trace", EgsIter * TM_MAX_TRACE),
                ("opta_trace_len", C.c_int32), ("opta_trace", OptaIter * (TM_MAX_TRACE + 1)),
                ("prep_ms", C.c_double)]


class StripPart(C.Structure):  # tm_strip_part
    _fields_ = [("best_rho", C.c_double), ("best_row", C.c_int32), ("best_col", C.c_int32),
                ("best_flags", C.c_int32), ("_pad0", C.c_int32), ("centers", C.c_int64),
                ("eliminated", C.c_int64), ("retained", C.c_int64),
                ("final_threshold", C.c_double)]


_P = C.c_void_p
_D = C.POINTER(C.c_double)
_U8 = C.POINTER(C.c_uint8)
_I = C.POINTER(C.c_int)

SIGNATURES = {
    "tm_last_error": (C.c_char_p, []),
    "tm_default_params": (None, [C.POINTER(MatchParams)]),
    "tm_ctx_create": (C.c_int, [C.c_int, C.POINTER(_P)]),
    "tm_ctx_destroy": (None, [_P]),
    "tm_ctx_synchronize": (C.c_int, [_P]),
    "tm_image_create_strip_u8": (C.c_int, [_P, C.c_int, C.c_int, C.c_int, C.c_int, _U8,
                                           C.POINTER(_P)]),
    "tm_image_upload_strip_u8": (C.c_int, [_P, _P, _U8]),
    "tm_image_sum_sq_rows": (C.c_int, [_P, _P, C.c_int, C.c_int, C.POINTER(C.c_uint64)]),
    "tm_image_set_noise_floor": (C.c_int, [_P, _P, C.c_uint64]),
    "tm_ctx_launch_count": (C.c_int64, [_P]),
    "tm_ctx_search_stats": (C.c_int, [_P, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "tm_ctx_split_stats": (C.c_int, [_P, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "tm_ctx_stream": (C.c_void_p, [_P]),
    "tm_ctx_set_profiling": (C.c_int, [_P, C.c_int]),
    "tm_ctx_phase_times": (C.c_int, [_P, C.c_char_p, C.c_size_t]),
    "tm_image_reset_cache": (C.c_int, [_P]),
    "tm_image_create": (C.c_int, [_P, _D, C.c_int, C.c_int, C.POINTER(_P)]),
    "tm_image_create_u8": (C.c_int, [_P, _U8, C.c_int, C.c_int, C.POINTER(_P)]),
    "tm_image_upload_u8": (C.c_int, [_P, _P, _U8]),
    "tm_image_download": (C.c_int, [_P, _P, _D]),
    "tm_image_is_integer": (C.c_int, [_P]),
    "tm_image_destroy": (None, [_P]),
    "tm_running_sum": (C.c_int, [_P, _P, C.c_int, C.c_int, _D]),
    "tm_window_stats": (C.c_int, [_P, _P, C.c_int, C.c_int, _D, _D, _U8]),
    "tm_brute_force_match": (C.c_int, [_P, _D, C.c_int, C.c_int, _P, C.POINTER(MatchResult),
                                       _D]),
    "tm_local_autocorrelation": (C.c_int, [_P, _P, C.c_int, C.c_int, C.c_int, C.c_int, _D]),
    "tm_autocorr_retained": (C.c_int, [_P, _P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                       C.POINTER(C.c_int64)]),
    "tm_efficient_group_size": (C.c_int, [_P, _P, C.c_int, C.c_int, C.c_int, C.c_int,
                                          C.c_double, C.c_double, C.c_int, _I, _I,
                                          C.POINTER(EgsIter), _I, _D]),
    "tm_blur": (C.c_int, [_P, _P, _D, C.c_int, _D]),
    "tm_blur_fidelity_map": (C.c_int, [_P, _P, _P, C.c_int, C.c_int, _D]),
    "tm_unblur_violations": (C.c_int, [_P, _P, _P, _D, C.c_int, C.c_int, C.c_double, _D,
                                       C.POINTER(C.c_int64)]),
    "tm_prepare": (C.c_int, [_P, _P, C.c_int, C.c_int, C.POINTER(MatchParams), C.POINTER(_P)]),
    "tm_prep_get_info": (C.c_int, [_P, C.POINTER(PrepInfo)]),
    "tm_prep_download": (C.c_int, [_P, _P, _D, _D]),
    "tm_prep_destroy": (None, [_P]),
    "tm_run": (C.c_int, [_P, _P, _P, _D, C.c_int, C.POINTER(MatchParams),
                         C.POINTER(MatchResult), _U8]),
    "tm_run_u8": (C.c_int, [_P, _P, _P, _U8, C.c_int, C.POINTER(MatchParams),
                            C.POINTER(MatchResult), _U8]),
    "tm_search": (C.c_int, [_P, _P, _D, C.c_int, C.c_int, C.POINTER(MatchParams),
                            C.POINTER(MatchResult)]),
    "tm_search_u8": (C.c_int, [_P, _P, _U8, C.c_int, C.c_int, C.POINTER(MatchParams),
                               C.POINTER(MatchResult)]),
    "tm_search_upload_u8": (C.c_int, [_P, _P, _U8, _U8, C.c_int, C.c_int,
                                      C.POINTER(MatchParams), C.POINTER(MatchResult)]),
    "tm_search_stream_u8": (C.c_int, [_P, C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_int,
                                      _U8, C.c_int, C.c_int, C.POINTER(MatchParams),
                                      C.POINTER(MatchResult)]),
    "tm_transitive_search": (C.c_int, [_P, _D, C.c_int, C.c_int, _P, _D, C.c_int, C.c_int,
                                       C.POINTER(MatchParams), C.POINTER(MatchResult), _U8]),
    "tm_transitive_search_ws": (C.c_int, [_P, _D, C.c_int, C.c_int, _P, _D, C.c_int, C.c_int,
                                          _D, _D, _U8, C.POINTER(MatchParams),
                                          C.POINTER(MatchResult), _U8]),
    "tm_center_scan": (C.c_int, [_P, _D, C.c_int, C.c_int, _P, C.c_int, C.c_int, _D, _U8, _I,
                                 _I, _D, _I]),
    "tm_refine_localization": (C.c_int, [_P, _D, C.c_int, C.c_int, _P, C.c_int, C.c_int,
                                         C.c_int, _I, _I, _D, _I]),
    "tm_match": (C.c_int, [_P, _D, C.c_int, C.c_int, _D, C.c_int, C.c_int,
                           C.POINTER(MatchParams), C.POINTER(MatchResult), _U8]),
    "tm_strip_autocorr": (C.c_int, [_P, _P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                    C.c_double, C.c_int, C.POINTER(C.c_int64)]),
    "tm_strip_commit": (C.c_int, [_P, _P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                  C.POINTER(MatchParams), C.POINTER(EgsIter), C.c_int,
                                  C.POINTER(_P)]),
    "tm_strip_search_begin": (C.c_int, [_P, _P, _P, _D, C.POINTER(MatchParams), C.c_int, C.c_int,
                                        _D]),
    "tm_strip_search_seed": (C.c_int, [_P, C.c_double, _D]),
    "tm_strip_fused_begin": (C.c_int, [_P, _P, _D, C.c_int, C.c_int, C.POINTER(MatchParams),
                                       C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int),
                                       C.POINTER(C.c_double)]),
    "tm_strip_fused_seed": (C.c_int, [_P, C.c_double, C.POINTER(C.c_double)]),
    "tm_strip_fused_egs": (C.c_int, [_P, C.c_double, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                     C.POINTER(C.c_int64)]),
    "tm_strip_fused_finish": (C.c_int, [_P, C.POINTER(StripPart)]),
    "tm_strip_search_finish": (C.c_int, [_P, C.c_double, C.POINTER(StripPart)]),
}


def header_symbols(path: str = HEADER) -> list:
    """Every function the C header declares (used by the CPU export test)."""
    text = open(path).read()
    return sorted(set(re.findall(r"\b(tm_[a-z0-9_]+)\s*\(", text)))


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1407_3535_b200.build` "
                "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int):
    if rc == TM_OK:
        return
    msg = lib().tm_last_error().decode()
    if rc == TM_EINVAL:
        raise InvalidArgument(msg)
    if rc == TM_ENODEV:
        raise NoDeviceError(msg)
    raise TmatchError(f"tmatch error {rc}: {msg}")
