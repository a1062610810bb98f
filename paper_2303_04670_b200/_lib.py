"""ctypes binding of libevconv.so (include/evconv.h).

There is no CPU fallback: importing an operator that needs the library
raises ``RuntimeError`` when the library or a CUDA device is missing.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

import torch

LIB_PATH = Path(__file__).resolve().parent / "libevconv.so"
ABI_VERSION = 3

ENC = {"count": 0, "timestamp": 1, "voxel": 2}
ACT = {"relu": 0, "sigmoid": 1, "tanh": 2, "leaky_relu": 3}


class EvcTensor(C.Structure):
    _fields_ = [
        ("vals", C.c_void_p),
        ("flags", C.c_void_p),
        ("vstride", C.c_int64),
        ("fstride", C.c_int64),
        ("C", C.c_int32),
        ("H", C.c_int32),
        ("W", C.c_int32),
        ("th", C.c_int32),
        ("tw", C.c_int32),
    ]


class EvcConvGeom(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("c_in", "c_out", "kh", "kw", "stride", "pad", "H", "W", "Ho", "Wo", "th", "tw")]


class EvcConvCfg(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("bn", "rh", "rw", "splits", "row", "thin", "drain")]


class EvcConvSparsify(C.Structure):
    _fields_ = [("hwc", C.c_void_p), ("hwc_stride", C.c_int64), ("cp", C.c_int32), ("pitch", C.c_int32),
                ("flags", C.c_void_p),
                ("fstride", C.c_int64), ("fany", C.c_void_p), ("partials", C.c_void_p)]


class EvcConvSubpixel(C.Structure):
    _fields_ = [("c_out", C.c_int32), ("Ho", C.c_int32), ("Wo", C.c_int32), ("reserved", C.c_int32),
                ("fany_in", C.c_void_p), ("border", C.c_void_p)]


class EvcMeterNode(C.Structure):
    _fields_ = [("part", C.c_void_p), ("n", C.c_int64), ("nflags", C.c_int64), ("dense", C.c_int64),
                ("c_out", C.c_int32), ("reserved", C.c_int32)]


class EvcSpNode(C.Structure):
    _fields_ = [("partials", C.c_void_p), ("n", C.c_int64), ("norm_ema", C.c_void_p), ("k", C.c_void_p),
                ("tp", C.c_double), ("decay", C.c_double)]


_P = C.c_void_p
_I32 = C.c_int32
_I64 = C.c_int64
_F = C.c_float
_D = C.c_double
_T = C.POINTER(EvcTensor)
_G = C.POINTER(EvcConvGeom)
_CF = C.POINTER(EvcConvCfg)
_SP = C.POINTER(EvcConvSparsify)
_SUB = C.POINTER(EvcConvSubpixel)

_PROTOS = {
    "evc_version": (_I32, []),
    "evc_last_error": (C.c_char_p, []),
    "evc_init": (_I32, []),
    "evc_set_pdl": (_I32, [_I32]),
    "evc_diff_mask": (_I32, [_P, _P, _I64, _T, _I32, _P]),
    "evc_make_tile_mask": (_I32, [_T, _I32, _P]),
    "evc_compact_scratch": (_I64, [_I64]),
    "evc_compact": (_I32, [_P, _I64, _P, _P, _P, _P]),
    "evc_count_flags": (_I32, [_T, _I32, _P, _P]),
    "evc_integrate": (_I32, [_P, _I64, _T, _I32, _P]),
    "evc_copy_masked": (_I32, [_T, _T, _I32, _P]),
    "evc_copy_dense": (_I32, [_P, _I64, _P, _I64, _I64, _I32, _P]),
    "evc_copy_bytes": (_I32, [_P, _I64, _P, _I64, _I64, _I32, _P]),
    "evc_conv_scatter_supported": (_I32, [_G]),
    "evc_conv_scatter_pack_len": (_I64, [_G]),
    "evc_conv_scatter_pack": (_I32, [_P, _G, _P]),
    "evc_conv_scatter_workspace": (_I64, [_G, _I32]),
    "evc_conv_scatter": (_I32, [_G, _T, _P, _T, _P, _I64, _I32, _I32, _P]),
    "evc_max_abs_diff": (_I32, [_P, _I64, _P, _I64, _I64, _I32, _P, _P]),
    "evc_conv_table_len": (_I64, [_G]),
    "evc_conv_table_fill": (_I32, [_G, _P]),
    "evc_conv_mask_scratch": (_I64, [_G, _I32]),
    "evc_conv_mask": (_I32, [_G, _T, _T, _P, _P, _P, _P, _P, _P, _P, _I32, _P]),
    "evc_hwc_channels": (_I32, [_I32]),
    "evc_to_hwc": (_I32, [_T, _P, _I64, _I32, _I32, _I32, _P]),
    "evc_conv_fused_supported": (_I32, [_G]),
    "evc_conv_fused_config": (_I32, [_G, _I32, _I32, _CF]),
    "evc_conv_fused_pack_len": (_I64, [_G, _CF]),
    "evc_conv_fused_pack": (_I32, [_P, _G, _CF, _P]),
    "evc_conv_fused_state_len": (_I64, [_G, _CF, _I32]),
    "evc_conv_fused_ctas": (_I64, [_G, _CF]),
    "evc_conv_fused": (_I32, [_G, _CF, _P, _I32, _I64, _P, _P, _T, _P, _P, _P, _P, _T, _I32, _F, _P, _I64, _T,
                              _SP, _I32, _I32, _P]),
    "evc_conv_fused_subpixel": (_I32, [_G, _CF, _P, _I32, _I64, _P, _P, _T, _P, _P, _P, _P, _T, _I32, _F, _P, _I64,
                                       _T, _SP, _SUB, _I32, _I32, _P]),
    "evc_subpixel_input_partials": (_I64, [_T, _I32]),
    "evc_subpixel_input": (_I32, [_T, _T, _P, _P, _I32, _I64, _I32, _P, _P, _I32, _P]),
    "evc_subpixel_border": (_I32, [_T, _P, _I32, _P, _I32, _P]),
    "evc_subpixel_input_border": (_I32, [_T, _T, _P, _P, _I32, _I64, _I32, _P, _P, _P, _I32, _P, _I32, _P]),
    "evc_tile_any": (_I32, [_T, _P, _I32, _P]),
    "evc_conv_trace": (_I32, [_P]),
    "evc_meter_step": (_I32, [_P, _I32, _I32, _P, _P, _P, _P, _P, _P, _I32, _P]),
    "evc_conv_workspace": (_I64, [_G, _I64, _I32]),
    "evc_conv_gemm": (_I32, [_G, _T, _P, _P, _P, _T, _P, _P, _P, _I32, _I32, _P, _P]),
    "evc_conv_tc_pack_len": (_I64, [_I32, _I64]),
    "evc_conv_tc_pack": (_I32, [_P, _I32, _I64, _P]),
    "evc_act_delta": (_I32, [_T, _P, _I64, _T, _I32, _F, _I32, _P]),
    "evc_act_dense": (_I32, [_P, _I64, _P, _I64, _P, _I64, _I64, _I32, _F, _I32, _P]),
    "evc_sparsify_partials": (_I64, [_T]),
    "evc_sparsify": (_I32, [_T, _P, _I64, _P, _T, _P, _P, _D, _D, _P, _P, _P, _I32, _I64, _I32, _P, _I32, _I32, _I32,
                            _P]),
    "evc_fold": (_I32, [_T, _P, _I64, _I32, _P]),
    "evc_upsample_sparsify_partials": (_I64, [_T]),
    "evc_upsample_sparsify": (_I32, [_T, _I32, _I32, _P, _I64, _P, _T, _P, _P, _D, _D, _P, _P, _P, _I32, _I64, _I32, _P,
                                     _I32,
                                     _I32, _I32, _P]),
    "evc_sparsify_finalize": (_I32, [_P, _I64, _P, _P, _D, _D, _I32, _I32, _P]),
    "evc_sumsq_dense": (_I32, [_P, _I64, _I64, _P, _I32, _I32, _P]),
    "evc_fill_segments": (_I32, [_P, _I32, _I32, _P]),
    "evc_add": (_I32, [_T, _T, _T, _I32, _P]),
    "evc_add_act": (_I32, [_T, _T, _P, _I64, _T, _I32, _F, _I32, _P]),
    "evc_mul": (_I32, [_T, _T, _P, _P, _I64, _T, _I32, _P]),
    "evc_binary_dense": (_I32, [_P, _I64, _P, _I64, _P, _I64, _I64, _I32, _I32, _P]),
    "evc_upsample": (_I32, [_T, _T, _I32, _I32, _I32, _P]),
    "evc_maxpool": (_I32, [_T, _P, _I64, _T, _I32, _I32, _I32, _I32, _P]),
    "evc_linear_workspace": (_I64, [_I32, _I64, _I32, _I32]),
    "evc_linear": (_I32, [_T, _P, _P, _T, _I32, _I32, _P, _P, _I32, _P]),
    "evc_bin_events_workspace": (_I64, [_I64, _I32, _I32, _I32]),
    "evc_bin_events": (_I32, [_P, _P, _P, _P, _I64, _I64, _I64, _I64, _I32, _I32, _I32, _I32, _P, _P, _I64, _P]),
    "evc_unpack_events": (_I32, [_P, _I64, _P, _P, _P, _P, _P]),
    "evc_count_increment": (_I32, [_P, _P, _P, _I64, _I64, _I64, _I64, _T, _P]),
    "evc_ingest_ring": (_I32, [_P, _P, _I64, _I64, _P, _P, _P, _P, _I32, _P]),
    "evc_encode_windows": (_I32, [_P, _P, _P, _P, _I64, _P, _I64, _I32, _I32, _I32, _P, _I64, _I32, _P]),
}

EXPORTED = tuple(_PROTOS)

_lock = threading.Lock()
_lib = None
_initialized = False


def load(require_cuda: bool = True):
    """Load and type the library; initialise its kernels when CUDA is up."""
    global _lib, _initialized
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_2303_04670_b200._build` "
                    "(there is no CPU fallback)")
            lib = C.CDLL(str(LIB_PATH))
            for name, (res, args) in _PROTOS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            if lib.evc_version() != ABI_VERSION:
                raise RuntimeError(f"libevconv ABI {lib.evc_version()} != {ABI_VERSION}")
            _lib = lib
        if require_cuda and not _initialized:
            if not torch.cuda.is_available():
                raise RuntimeError("paper_2303_04670_b200 needs a CUDA device (B200); there is no CPU fallback")
            torch.cuda.init()
            check(_lib.evc_init(), "evc_init")
            import os
            _lib.evc_set_pdl(1 if os.environ.get("EVC_PDL", "0") == "1" else 0)
            _initialized = True
        return _lib


def lib():
    return _lib if (_lib is not None and _initialized) else load()


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = _lib.evc_last_error().decode(errors="replace") if _lib is not None else ""
        raise RuntimeError(f"libevconv {what} failed ({rc}): {msg}")


def stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t) -> int | None:
    return None if t is None else int(t.data_ptr())


def tdesc(vals, flags, vstride, fstride, c, h, w, th, tw) -> EvcTensor:
    return EvcTensor(vals, flags, int(vstride), int(fstride), int(c), int(h), int(w), int(th), int(tw))
