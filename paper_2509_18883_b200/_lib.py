"""ctypes binding of the C ABI declared in include/rlk.h (`_rlk.so`, built by `_build.py`).

There is no fallback: if the library is missing or fails to load, every entry point raises.
Device buffers are passed as raw pointers (`tensor.data_ptr()`), streams as `cudaStream_t` handles.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

RLK_OK = 0
RLK_ERR_INVALID = -1
RLK_ERR_CUDA = -2
RLK_ERR_UNSUPPORTED = -3

RLK_BF16, RLK_F32, RLK_F64 = 0, 1, 2
RLK_MERGE_WS_HEADER = 4096  # include/rlk.h
RLK_MAX_EXPERTS = 8
RLK_FUSION_ITEM = 65536

LIB_PATH = Path(os.environ.get("RLK_LIB_PATH", Path(__file__).resolve().parent / "_rlk.so"))

# Layout of rlk_fusion_segment (include/rlk.h): 104 bytes, 8-byte aligned.
SEGMENT_DTYPE = np.dtype([
    ("base", "<u8"), ("expert", "<u8", (RLK_MAX_EXPERTS,)), ("out", "<u8"),
    ("numel", "<u8"), ("j0", "<u8"), ("tensor", "<u4"), ("item0", "<u4"),
])
assert SEGMENT_DTYPE.itemsize == 104


class FusionPlanC(C.Structure):
    _fields_ = [("segs", C.c_void_p), ("seg_item_prefix", C.c_void_p), ("n_segs", C.c_uint32),
                ("n_items", C.c_uint32)]


class ClipC(C.Structure):
    _fields_ = [("eps_neg_low", C.c_double), ("eps_pos_high", C.c_double), ("eps_neg_high", C.c_double),
                ("tis_cap", C.c_double), ("guard_positive", C.c_int32)]


_P = C.c_void_p
_U64 = C.c_uint64
_I = C.c_int
_D = C.c_double

# name -> (restype, argtypes); every symbol declared in include/rlk.h
SIGNATURES = {
    "rlk_last_error": (C.c_char_p, []),
    "rlk_abi_version": (_I, []),
    "rlk_device_sm_count": (_I, [_I]),
    "rlk_fusion_sumsq": (_I, [C.POINTER(FusionPlanC), _I, _I, _I, _P, _P, _I, _P, _U64, _P, _U64, _P]),
    "rlk_fusion_finalize": (_I, [_P, _P, C.c_uint32, _I, _I, _D, _P, _P, _P, _P]),
    "rlk_fusion_mask_bitmap": (_I, [_P, _I, _U64, _U64, _P, _U64, _P]),
    "rlk_fusion_mask_bitmap_range": (_I, [_P, _I, _U64, _U64, _U64, _P, _U64, _P]),
    "rlk_fusion_merge": (_I, [C.POINTER(FusionPlanC), _I, _I, _I, _I, _P, _P, _I, _P, _U64, _D, _P, _U64, _I,
                              _P, _I, _P]),
    "rlk_fusion_merge_ws": (_I, [C.POINTER(FusionPlanC), _I, _I, _I, _I, _P, _P, _I, _P, _U64, _D, _P, _U64, _I,
                                 _P, _I, _P, _U64, _P]),
    "rlk_grpo_fwd": (_I, [_P, _I, _U64, _U64, _U64, _P, _P, _P, _P, _P, _P, _P, _P, _P, C.POINTER(ClipC), _P, _P,
                          _P, _P, _P, _P, _U64, _P]),
    "rlk_segment_sum_f64": (_I, [_P, _P, _U64, _P, _P]),
    "rlk_grpo_fused_bf16": (_I, [_P, _U64, _U64, _U64, _P, _P, _P, _P, _P, _P, _P, _P, _P, C.POINTER(ClipC), _D,
                                 _P, _P, _P, _P, _P, _P, _U64, _P]),
    "rlk_grpo_fused": (_I, [_P, _I, _U64, _U64, _U64, _P, _P, _P, _P, _P, _P, _P, _P, _P, C.POINTER(ClipC), _D,
                            _P, _P, _P, _P, _P, _P, _U64, _P]),
    "rlk_grpo_bwd": (_I, [_P, _I, _U64, _U64, _U64, _P, _P, _P, _P, _P, _P, _P, _P, _I, _U64, _P]),
    "rlk_logsoftmax_rows": (_I, [_P, _I, _U64, _U64, _U64, _P, _P, _P, _I, _P]),
    "rlk_nonfinite_count": (_I, [_P, _I, _U64, _P, _P]),
    "rlk_scaled_add": (_I, [_P, _P, _D, _P, _I, _U64, _P]),
    "rlk_synth_normal": (_I, [_P, _I, _U64, _U64, _U64, _D, _P, _P]),
    "rlk_checksum64": (_I, [_P, _U64, _U64, _P, _P]),
    "rlk_loader_create": (_P, [_U64, _I, _I]),
    "rlk_loader_destroy": (None, [_P]),
    "rlk_loader_last_error": (C.c_char_p, []),
    "rlk_loader_h2d": (_I, [_P, _P, _P, _U64, _P]),
    "rlk_loader_d2h": (_I, [_P, _P, _P, _U64, _P]),
    "rlk_loader_synth_h2d": (_I, [_P, _P, _I, _U64, _U64, _U64, _D, _U64, _D, _P]),
    "rlk_loader_d2h_checksum": (_I, [_P, _P, _U64, C.POINTER(C.c_uint64), _P]),
}

_lib = None


class RlkError(RuntimeError):
    pass


def lib() -> C.CDLL:
    """Load `_rlk.so` (building it first if RLK_AUTOBUILD=1). Raises if it cannot be loaded."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists() and os.environ.get("RLK_AUTOBUILD", "0") == "1":
        from ._build import build
        build()
    if not LIB_PATH.exists():
        raise RlkError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                       "(there is no CPU fallback)")
    handle = C.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(handle, name, None)
        if fn is None:
            continue
        fn.restype = res
        fn.argtypes = args
    _lib = handle
    return handle


def check(status: int, where: str = "") -> None:
    """Map a C-ABI status to the reference's exception types."""
    if status == RLK_OK:
        return
    msg = lib().rlk_last_error().decode(errors="replace")
    if status == RLK_ERR_INVALID:
        raise ValueError(msg or where)
    raise RlkError(f"{where}: {msg} (status {status})")


def call(name: str, *args) -> None:
    """One C-ABI entry point, inside an NVTX range of its name (visible in Nsight timelines; a no-op
    marker without a profiler attached)."""
    nv = _nvtx()
    if nv is None:
        check(getattr(lib(), name)(*args), name)
        return
    nv.range_push(name)
    try:
        check(getattr(lib(), name)(*args), name)
    finally:
        nv.range_pop()


_NVTX = None


def _nvtx():
    global _NVTX
    if _NVTX is None:
        try:
            import torch
            _NVTX = torch.cuda.nvtx if torch.cuda.is_available() else False
        except Exception:  # pragma: no cover - torch without CUDA
            _NVTX = False
    return _NVTX or None


class nvtx_range:
    """`with nvtx_range("rlk.fusion_step"):` -- an NVTX range around a multi-kernel step."""

    def __init__(self, name: str):
        self.name = name

    def __enter__(self):
        nv = _nvtx()
        if nv is not None:
            nv.range_push(self.name)
        return self

    def __exit__(self, *exc):
        nv = _nvtx()
        if nv is not None:
            nv.range_pop()
        return False


def dtype_code(dtype) -> int:
    import torch
    if dtype == torch.bfloat16:
        return RLK_BF16
    if dtype == torch.float32:
        return RLK_F32
    if dtype == torch.float64:
        return RLK_F64
    raise ValueError(f"unsupported dtype {dtype} (bf16, f32, f64)")


def stream_handle(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()
