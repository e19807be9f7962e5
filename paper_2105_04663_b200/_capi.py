"""ctypes binding of ``include/spmd_b200.h`` (the C ABI).

This is the binding a maintainer of the reference would add (see
INTEGRATION.md): plain pointers, sizes and a stream handle; torch is only
used by the caller to own device memory.  Loading fails loudly when the
library has not been built -- there is no CPU fallback anywhere.
"""

from __future__ import annotations

import ctypes
import os
from typing import Sequence

from .ir import DType

MAX_RANK = 8
_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib",
                         "libspmd_b200.so")

DTYPE_CODE = {DType.F32: 0, DType.S32: 1, DType.U32: 2, DType.PRED: 3, DType.BF16: 4}

OK, ERR_INVALID, ERR_SHAPE, ERR_SUBGROUP, ERR_DIV_ZERO, ERR_CUDA, ERR_NCCL, \
    ERR_UNSUPPORTED = range(8)


class SpmdTensor(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("dtype", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("dims", ctypes.c_int64 * MAX_RANK)]


class SpmdDotDims(ctypes.Structure):
    _fields_ = [("n_batch", ctypes.c_int32), ("n_contract", ctypes.c_int32),
                ("lhs_batch", ctypes.c_int32 * MAX_RANK),
                ("rhs_batch", ctypes.c_int32 * MAX_RANK),
                ("lhs_contracting", ctypes.c_int32 * MAX_RANK),
                ("rhs_contracting", ctypes.c_int32 * MAX_RANK),
                ("epilogue", ctypes.c_int32)]


class SpmdConvDims(ctypes.Structure):
    _fields_ = [("lhs_batch", ctypes.c_int32), ("lhs_feature", ctypes.c_int32),
                ("rhs_in_feature", ctypes.c_int32), ("rhs_out_feature", ctypes.c_int32),
                ("out_batch", ctypes.c_int32), ("out_feature", ctypes.c_int32),
                ("n_spatial", ctypes.c_int32)] + \
        [(n, ctypes.c_int32 * MAX_RANK) for n in (
            "lhs_spatial", "rhs_spatial", "out_spatial", "size", "stride", "pad_low",
            "pad_high", "base_dilation", "window_dilation")] + [("epilogue", ctypes.c_int32)]


_T = SpmdTensor
_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
_PI32 = ctypes.POINTER(ctypes.c_int32)
_PI64 = ctypes.POINTER(ctypes.c_int64)

_SIGNATURES = {
    "spmd_version": ([], ctypes.c_char_p),
    "spmd_status_string": ([_I], ctypes.c_char_p),
    "spmd_last_error": ([], ctypes.c_char_p),
    "spmd_check_device_errors": ([_P], _I),
    "spmd_launch_count": ([], _I64),
    "spmd_set_sm_limit": ([_I], _I),
    "spmd_set_option": ([ctypes.c_char_p, _I64], _I),
    "spmd_get_option": ([ctypes.c_char_p, _PI64], _I),
    "spmd_iota": ([_T, _I, _I64, _P], _I),
    "spmd_partition_id": ([_T, _I64, ctypes.c_int32, _P], _I),
    "spmd_constant": ([_T, _T, _I64, _P], _I),
    "spmd_unary": ([_I, _T, _T, _I64, _P], _I),
    "spmd_binary": ([_I, _I, _T, _T, _T, _I64, _P], _I),
    "spmd_select": ([_T, _T, _T, _T, _I64, _P], _I),
    "spmd_convert": ([_T, _T, _I64, _P], _I),
    "spmd_broadcast": ([_T, _T, _PI32, _I64, _P], _I),
    "spmd_transpose": ([_T, _T, _PI32, _I64, _P], _I),
    "spmd_transpose_relu": ([_T, _T, _PI32, _I64, _P], _I),
    "spmd_reverse": ([_T, _T, _PI32, _I, _I64, _P], _I),
    "spmd_pad": ([_T, _T, _T, _PI64, _PI64, _PI64, _I64, _P], _I),
    "spmd_slice": ([_T, _T, _PI64, _PI64, _I64, _P], _I),
    "spmd_dynamic_slice": ([_T, ctypes.POINTER(_T), _T, _I64, _P], _I),
    "spmd_dynamic_update_slice": ([_T, _T, ctypes.POINTER(_T), _T, _I64, _P], _I),
    "spmd_concat": ([ctypes.POINTER(_T), _I, _I, _T, _I64, _P], _I),
    "spmd_rotate": ([_T, _T, _I, _I64, _I64, _P], _I),
    "spmd_shift": ([_T, _T, _T, _I, _I64, _I64, _P], _I),
    "spmd_reduce": ([_T, _T, _T, _PI32, _I, _I, _I64, _P], _I),
    "spmd_dot": ([_T, _T, _T, ctypes.POINTER(SpmdDotDims), _I64, _P], _I),
    "spmd_dot_add": ([_T, _T, _T, _T, ctypes.POINTER(SpmdDotDims), _I64, _P], _I),
    "spmd_convolution": ([_T, _T, _T, ctypes.POINTER(SpmdConvDims), _I64, _P], _I),
    "spmd_softmax_lastdim": ([_T, _T, _I64, _P], _I),
    "spmd_softmax_backward_lastdim": ([_T, _T, _T, _I64, _P], _I),
    "spmd_relu_backward": ([_T, _T, _T, _I64, _P], _I),
    "spmd_attention": ([_T, _T, _T, _T, ctypes.c_float, _I64, _P], _I),
    "spmd_attention_layout": ([_T, _T, _T, _T, ctypes.c_float, _I, _I64, _P], _I),
    "spmd_mask_range": ([_T, _T, _T, _T, _I, _I64, _I64, _I, _I64, _P], _I),
    "spmd_halo_window": ([ctypes.POINTER(_T), _I, _I, _T, _I, _T, _T, _I64, _I64, _I, _T, _I64,
                          _P], _I),
    "spmd_halo_convolution": ([ctypes.POINTER(_T), _I, _I, _T, _I, _T, _I64, _I64, _I, _T, _T,
                               _T, ctypes.POINTER(SpmdConvDims), _I64, _P], _I),
    "spmd_gemm_bf16": ([_P, _P, _P, _I64, _I64, _I64, _I, _P], _I),
    "spmd_moe_route": ([_T, _I, _T, _T, _T, _I64, _P], _I),
    "spmd_moe_dispatch": ([_T, _T, _T, _T, _I64, _P], _I),
    "spmd_moe_combine": ([_T, _T, _T, _T, _T, _I64, _P], _I),
    "spmd_moe_dispatch_ex": ([_T, _T, _T, _T, _I, _I64, _P], _I),
    "spmd_moe_combine_ex": ([_T, _T, _T, _T, _T, _I, _I64, _P], _I),
    "spmd_moe_masks": ([_T, _T, _T, _T, _T, _I64, _P], _I),
    "spmd_local_all_gather": ([_T, _T, _I, _PI32, _I, _I, _I64, _P], _I),
    "spmd_local_all_gather_split": ([_T, _T, _T, _I, _PI32, _I, _I, _I64, _P], _I),
    "spmd_local_all_gather_split_t": ([_T, _T, _T, _PI32, _I, _I, _I64, _P], _I),
    "spmd_dot_f32_presplit": ([_T, _T, _T, _T, _T, _T, _T, ctypes.POINTER(SpmdDotDims), _I64,
                               _P], _I),
    "spmd_local_all_reduce": ([_T, _T, _I, _PI32, _I, _I, _I64, _P], _I),
    "spmd_local_reduce_scatter": ([_T, _T, _I, _I, _PI32, _I, _I, _I64, _P], _I),
    "spmd_local_all_to_all": ([_T, _T, _I, _I, _PI32, _I, _I, _I64, _P], _I),
    "spmd_local_collective_permute": ([_T, _T, _PI32, _I, _I64, _P], _I),
    "spmd_comm_id_bytes": ([], _I),
    "spmd_comm_get_unique_id": ([_P], _I),
    "spmd_comm_init": ([ctypes.POINTER(_P), _I, _I, _P], _I),
    "spmd_comm_destroy": ([_P], _I),
    "spmd_comm_set_workspace": ([_P, _P, _I64], _I),
    "spmd_all_gather": ([_P, _T, _T, _I, _PI32, _I, _I, _P], _I),
    "spmd_all_reduce": ([_P, _T, _T, _I, _PI32, _I, _I, _P], _I),
    "spmd_reduce_scatter": ([_P, _T, _T, _I, _I, _PI32, _I, _I, _P], _I),
    "spmd_all_to_all": ([_P, _T, _T, _I, _I, _PI32, _I, _I, _P], _I),
    "spmd_collective_permute": ([_P, _T, _T, _PI32, _I, _P], _I),
    "spmd_comm_enable_peer": ([_P, _I64, _P], _I),
    "spmd_comm_peer_bytes": ([_P], _I64),
    "spmd_comm_reserve_fused": ([_P, _I64], _I),
    "spmd_comm_fused_half": ([_P], _I64),
    "spmd_dot_reduce_scatter": ([_P, _T, _T, _T, ctypes.POINTER(SpmdDotDims), _I, _PI32, _I, _I,
                                 _P], _I),
    "spmd_dot_reduce_scatter_add": ([_P, _T, _T, _T, _T, ctypes.POINTER(SpmdDotDims), _I, _PI32,
                                     _I, _I, _P], _I),
    "spmd_dot_all_to_all": ([_P, _T, _T, _T, ctypes.POINTER(SpmdDotDims), _I, _I, _PI32, _I, _I,
                             _P], _I),
    "spmd_moe_dispatch_all_to_all": ([_P, _T, _T, _T, _T, _T, _PI32, _I, _I, _P], _I),
    "spmd_peer_all_gather": ([_P, _T, _T, _I, _PI32, _I, _I, _I64, _I, _I, _P], _I),
    "spmd_peer_stage": ([_P, _T, _I64, _P], _I),
    "spmd_peer_barrier": ([_P, _I, _P], _I),
    "spmd_peer_all_to_all": ([_P, _T, _T, _I, _I, _PI32, _I, _I, _I64, _I, _P], _I),
    "spmd_peer_push_all_gather": ([_P, _T, _T, _I, _PI32, _I, _I, _I64, _I, _P], _I),
    "spmd_comm_heap_ptr": ([_P, _I64], ctypes.c_void_p),
    "spmd_peer_collective_permute": ([_P, _T, _T, _PI32, _I, _I64, _I, _P], _I),
    "spmd_peer_slice_collective_permute": ([_P, _T, _I, _I64, _T, _PI32, _I, _I64, _I, _P], _I),
}

_lib = None


def library_path() -> str:
    return _LIB_PATH


def exported_symbols() -> list[str]:
    return sorted(_SIGNATURES)


def lib():
    """The loaded C library (raises if it was never built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(
                f"{_LIB_PATH} is missing: build it with "
                "`python paper_2105_04663_b200/csrc/build.py` (there is no CPU path)")
        # torch first, so its NCCL (the one we link) is already resident.
        import torch  # noqa: F401
        l = ctypes.CDLL(_LIB_PATH)
        for name, (args, res) in _SIGNATURES.items():
            f = getattr(l, name)
            f.argtypes = args
            f.restype = res
        _lib = l
    return _lib


class SpmdError(Exception):
    def __init__(self, status: int, fn: str, msg: str):
        self.status = status
        super().__init__(f"{fn}: {msg}")


def check(status: int, fn: str = "spmd") -> None:
    if status == OK:
        return
    l = lib()
    msg = (l.spmd_last_error() or b"").decode() or l.spmd_status_string(status).decode()
    from . import executor as ex
    if status == ERR_DIV_ZERO:
        raise ex.DivideByZero(msg)
    if status == ERR_SUBGROUP:
        raise ex.SubgroupMismatch(msg)
    if status in (ERR_INVALID, ERR_SHAPE, ERR_UNSUPPORTED):
        raise ex.EvalError(f"{fn}: {msg}")
    raise SpmdError(status, fn, msg)


def set_option(name: str, value: int) -> None:
    """spmd_set_option: switch a kernel variant / tuning knob at run time."""
    check(lib().spmd_set_option(name.encode(), int(value)), "spmd_set_option")


def get_option(name: str) -> int:
    v = ctypes.c_int64()
    check(lib().spmd_get_option(name.encode(), ctypes.byref(v)), "spmd_get_option")
    return v.value


class option:
    """Context manager: ``with option("gemm_mode", 2): ...`` restores the
    previous value on exit."""

    def __init__(self, name: str, value: int):
        self.name, self.value = name, value

    def __enter__(self):
        self.old = get_option(self.name)
        set_option(self.name, self.value)
        return self

    def __exit__(self, *exc):
        set_option(self.name, self.old)
        return False


def i32_array(vals: Sequence[int]):
    vals = [int(v) for v in vals]
    return (ctypes.c_int32 * max(1, len(vals)))(*vals)


def i64_array(vals: Sequence[int]):
    vals = [int(v) for v in vals]
    return (ctypes.c_int64 * max(1, len(vals)))(*vals)
