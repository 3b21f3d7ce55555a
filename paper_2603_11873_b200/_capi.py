"""ctypes binding of the C ABI declared in include/adafuse_b200.h.

This is the only module that touches ``libadafuse_b200.so``.  There is NO fallback: if the
library is missing or no CUDA device is present, the product path raises ``DeviceError``.
"""

from __future__ import annotations

import ctypes
import os

from . import errors

HERE = os.path.dirname(os.path.abspath(__file__))
# AF_LIB_PATH: an alternative build of the same library (kernel-variant A/B runs on one box)
LIB_PATH = os.environ.get("AF_LIB_PATH") or os.path.join(HERE, "libadafuse_b200.so")

AF_ABI_VERSION = 3
AF_OK, AF_EVALUE, AF_EDIM, AF_EPRECISION, AF_EALIAS, AF_EINPUT, AF_ESTATE, AF_EINDEX, AF_ECUDA = range(9)
AF_BF16, AF_F32 = 0, 1
AF_SWITCH_INPLACE, AF_SWITCH_FROM_PRISTINE = 0, 1
AF_COMPUTE_AUTO, AF_COMPUTE_EXACT, AF_COMPUTE_FMA, AF_COMPUTE_MMA = 0, 1, 2, 3
AF_MAX_K = 8
AF_EPI_NONE, AF_EPI_GELU_RESIDUAL, AF_EPI_RESIDUAL = 0, 1, 2

COMPUTE_MODES = {"auto": AF_COMPUTE_AUTO, "exact": AF_COMPUTE_EXACT, "fma": AF_COMPUTE_FMA, "mma": AF_COMPUTE_MMA}

_STATUS_TO_EXC = {
    AF_EVALUE: ValueError,
    AF_EDIM: errors.DimensionError,
    AF_EPRECISION: errors.PrecisionError,
    AF_EALIAS: errors.AliasingError,
    AF_EINPUT: errors.InputError,
    AF_ESTATE: errors.StateError,
    AF_EINDEX: IndexError,
    AF_ECUDA: errors.DeviceError,
}


class Decision(ctypes.Structure):
    """`af_decision`: routing.py:37-46 `GateDecision` as a 128-byte POD."""

    _fields_ = [
        ("k", ctypes.c_int32),
        ("ids", ctypes.c_int32 * AF_MAX_K),
        ("weights", ctypes.c_float * AF_MAX_K),
        ("reserved", ctypes.c_int32 * 15),
    ]


class SegmentDesc(ctypes.Structure):
    """`af_segment_desc`: linalg.py:183-217 `Segment` as addresses."""

    _fields_ = [
        ("target", ctypes.c_void_p),
        ("pristine", ctypes.c_void_p),
        ("down", ctypes.c_void_p),
        ("up", ctypes.c_void_p),
        ("d_out", ctypes.c_int32),
        ("d_in", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("n_experts", ctypes.c_int32),
        ("ld_target", ctypes.c_int64),
        ("ld_down", ctypes.c_int64),
        ("ld_up", ctypes.c_int64),
        ("down_expert_stride", ctypes.c_int64),
        ("up_expert_stride", ctypes.c_int64),
    ]


class GemvPhase(ctypes.Structure):
    """`af_gemv_phase`: one projection of a chained switch + GEMV launch."""

    _fields_ = [
        ("xin", ctypes.c_void_p),
        ("acc_in", ctypes.c_void_p),
        ("res", ctypes.c_void_p),
        ("h_out", ctypes.c_void_p),
        ("norm_w", ctypes.c_void_p),
        ("acc_out", ctypes.c_void_p),
        ("eps", ctypes.c_float),
        ("prologue", ctypes.c_int32),
        ("inv_out", ctypes.c_void_p),
        ("inv_in", ctypes.c_void_p),
    ]


class GvPhase(ctypes.Structure):
    """`af_gv_phase`: one projection of a chained plain-GEMV launch."""

    _fields_ = [
        ("w", ctypes.c_void_p),
        ("rows", ctypes.c_int32),
        ("cols", ctypes.c_int32),
        ("ld", ctypes.c_int64),
        ("x", ctypes.c_void_p),
        ("out", ctypes.c_void_p),
        ("res", ctypes.c_void_p),
        ("norm_w", ctypes.c_void_p),
        ("eps", ctypes.c_float),
        ("prologue", ctypes.c_int32),
        ("epilogue", ctypes.c_int32),
    ]


class FwPhase(ctypes.Structure):
    """`af_fw_phase`: one record of the persistent forward's device-side phase table."""

    _fields_ = [
        ("w", ctypes.c_void_p),
        ("x", ctypes.c_void_p),
        ("out", ctypes.c_void_p),
        ("res", ctypes.c_void_p),
        ("norm_w", ctypes.c_void_p),
        ("k_cache", ctypes.c_void_p),
        ("v_cache", ctypes.c_void_p),
        ("ld", ctypes.c_int64),
        ("rows", ctypes.c_int32),
        ("cols", ctypes.c_int32),
        ("eps", ctypes.c_float),
        ("prologue", ctypes.c_int32),
        ("epilogue", ctypes.c_int32),
        ("kind", ctypes.c_int32),
    ]


AF_FW_GEMV, AF_FW_ATTN_PARTIAL, AF_FW_ATTN_COMBINE = 0, 1, 2

assert ctypes.sizeof(Decision) == 128

_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_f32 = ctypes.c_float

# name -> (restype, argtypes); every symbol include/adafuse_b200.h declares
SIGNATURES = {
    "af_abi_version": (ctypes.c_int, []),
    "af_last_error": (ctypes.c_char_p, []),
    "af_device_info": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)] * 3 + [ctypes.POINTER(_i64)]),
    "af_launch_count": (_i64, []),
    "af_last_switch_kernel": (ctypes.c_char_p, []),
    "af_set_pdl": (ctypes.c_int, [_i32]),
    "af_set_gemv_variant": (ctypes.c_int, [_i32, _i32]),
    "af_set_umma": (ctypes.c_int, [_i32]),
    "af_set_umma_pieces": (ctypes.c_int, [_i32]),
    "af_table_create": (ctypes.c_int, [ctypes.POINTER(SegmentDesc), _i32, _i32, _i32, ctypes.POINTER(_vp)]),
    "af_table_destroy": (ctypes.c_int, [_vp]),
    "af_table_info": (ctypes.c_int, [_vp, ctypes.POINTER(_i32), ctypes.POINTER(_i64), ctypes.POINTER(_i32), ctypes.POINTER(_i32)]),
    "af_table_status": (ctypes.c_int, [_vp, _vp]),
    "af_table_set_error_word": (ctypes.c_int, [_vp, _vp]),
    "af_flag_message": (ctypes.c_char_p, [_i32]),
    "af_pregate": (ctypes.c_int, [_vp, _i32, _i32, _i32, _vp, _i32, _vp, _i32, _vp, _vp, _vp]),
    "af_fused_switch": (ctypes.c_int, [_vp, _vp, _vp, ctypes.POINTER(Decision), ctypes.POINTER(Decision), _i32, _f32, _i32, _i32, _vp]),
    "af_merge": (ctypes.c_int, [_vp, _vp, ctypes.POINTER(Decision), _i32, _f32, _i32, _vp]),
    "af_unmerge": (ctypes.c_int, [_vp, _vp, ctypes.POINTER(Decision), _i32, _f32, _i32, _vp]),
    "af_sgmm": (ctypes.c_int, [_vp, _i32, _i32, _vp]),
    "af_refresh_from_pristine": (ctypes.c_int, [_vp, _vp]),
    "af_max_deviation": (ctypes.c_int, [_vp, _vp, _vp]),
    "af_gemv": (ctypes.c_int, [_vp, _i32, _i32, _i32, _i64, _vp, _vp, _i32, _vp, _vp]),
    "af_gemv_t": (ctypes.c_int, [_vp, _i32, _i32, _i32, _i64, _vp, _vp, _vp]),
    "af_argmax": (ctypes.c_int, [_vp, _i32, _vp, _vp]),
    "af_embed": (ctypes.c_int, [_vp, _i32, _i32, _vp, _vp, _vp]),
    "af_gemv_fused": (ctypes.c_int, [_vp, _i32, _i32, _i64, _vp, _vp, _i32, _vp, _f32, _i32, _vp, _vp]),
    "af_attn_decode": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp]),
    "af_argmax_val": (ctypes.c_int, [_vp, _i32, _i32, _vp, _vp, _vp]),
    "af_step_advance": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _vp, _i32, _vp]),
    "af_group_create": (ctypes.c_int, [_vp, ctypes.POINTER(_i32), _i32, ctypes.POINTER(_vp)]),
    "af_group_destroy": (ctypes.c_int, [_vp]),
    "af_chain_create": (ctypes.c_int, [_vp, ctypes.POINTER(_i32), ctypes.POINTER(_i32), _i32, ctypes.POINTER(_vp)]),
    "af_chain_create_weighted": (ctypes.c_int, [_vp, ctypes.POINTER(_i32), ctypes.POINTER(_i32), _i32, ctypes.POINTER(_f32), _i32, ctypes.POINTER(_vp)]),
    "af_group_info": (ctypes.c_int, [_vp, ctypes.POINTER(_i32), ctypes.POINTER(_i32), ctypes.POINTER(_i32), ctypes.POINTER(_i32), ctypes.POINTER(_i32), ctypes.POINTER(_i64)]),
    "af_switch_gemv_chain": (ctypes.c_int, [_vp, _vp, _vp, _i32, _f32, _i32, ctypes.POINTER(GemvPhase), _i32, _vp, _i32, _vp]),
    "af_switch_gemv": (ctypes.c_int, [_vp, _vp, _vp, _i32, _f32, _i32, _vp, _vp, _vp, _vp, _i32, _vp, _f32, _vp, _i32, _vp]),
    "af_gemv_chain": (ctypes.c_int, [ctypes.POINTER(GvPhase), _i32, _vp, _vp, _i32, _vp]),
    "af_forward_validate": (ctypes.c_int, [ctypes.POINTER(FwPhase), _i32, _i32, _i32, _i32, ctypes.POINTER(_i32)]),
    "af_forward_persistent": (ctypes.c_int, [_vp, _i32, _i32, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _i32, _vp]),
    "af_plan_build": (ctypes.c_int, [_vp, _vp, _vp, _i32, _f32, _i32, _vp]),
    "af_set_timeline": (ctypes.c_int, [_vp, _i32, _i64]),
    "af_accum_to_f32": (ctypes.c_int, [_vp, _vp, _vp, _i32, _vp]),
    "af_group_set_peers": (ctypes.c_int, [_vp, _i32, ctypes.POINTER(ctypes.c_int64), _i32]),
    "af_peer_barrier": (ctypes.c_int, [_vp, _vp, _i32, ctypes.POINTER(ctypes.c_int64), _vp, _vp]),
    "af_peer_wait": (ctypes.c_int, [_vp, _i32, _vp, _vp]),
    "af_peer_bcast": (ctypes.c_int, [_vp, _vp, _vp, _i32, _i32, _vp, _vp, _i32, ctypes.POINTER(ctypes.c_int64), _vp, _vp]),
    "af_peer_argmax": (ctypes.c_int, [_vp, _vp, _vp, _i32, _vp, _vp, _i32, ctypes.POINTER(ctypes.c_int64), _vp, _vp, _vp]),
    "af_attn_decode_fix": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp]),
}
AF_FIX_SHIFT = 40
AF_TIMELINE_SLOTS = 42
AF_CHAIN_PDL, AF_CHAIN_PLAN_PREBUILT = 1, 2
AF_PRO_NONE, AF_PRO_RMSNORM, AF_PRO_SILU_MUL, AF_PRO_RMSNORM_DEFERRED = 0, 1, 2, 3

_lib = None


def lib():
    """The loaded C-ABI library.  Raises DeviceError when it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise errors.DeviceError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)"
            )
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.af_abi_version() != AF_ABI_VERSION:
            raise errors.DeviceError("libadafuse_b200.so ABI version mismatch; rebuild it")
        _lib = L
    return _lib


def check(status: int) -> None:
    """Map a C-ABI status to the reference's exception classes (errors.py)."""
    if status == AF_OK:
        return
    msg = lib().af_last_error().decode("utf-8", "replace")
    raise _STATUS_TO_EXC.get(status, errors.DeviceError)(msg)


def raise_for_flag(flag: int) -> None:
    """Raise the reference's exception class for a status word a kernel raised on the device
    (the asynchronous form of `af_table_status`; include/adafuse_b200.h af_table_set_error_word)."""
    if flag == AF_OK:
        return
    msg = lib().af_flag_message(int(flag)).decode("utf-8", "replace")
    raise _STATUS_TO_EXC.get(int(flag), errors.DeviceError)(msg)


def require_cuda():
    """torch with a visible CUDA device, or DeviceError -- never a silent CPU path."""
    import torch

    if not torch.cuda.is_available():
        raise errors.DeviceError("no CUDA device visible: the AdaFuse B200 path has no CPU fallback")
    return torch


def stream_ptr() -> int:
    """The cudaStream_t of torch's current stream (all launches go there)."""
    import torch

    return torch.cuda.current_stream().cuda_stream


def launch_count() -> int:
    return int(lib().af_launch_count())


def device_info() -> dict:
    sm, maj, minor, l2 = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), _i64()
    check(lib().af_device_info(ctypes.byref(sm), ctypes.byref(maj), ctypes.byref(minor), ctypes.byref(l2)))
    return {"sm_count": sm.value, "cc": (maj.value, minor.value), "l2_bytes": l2.value}
