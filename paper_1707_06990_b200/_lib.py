"""ctypes binding of libdpb.so (include/dpb.h).

The library is built in-tree (``python -m paper_1707_06990_b200.build``) and
loaded from ``paper_1707_06990_b200/_build/libdpb.so``.  There is no fallback:
if the library is missing, importing the binding raises.
"""
from __future__ import annotations

import ctypes as C
import os

from . import errors

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "_build", "libdpb.so")

_P = C.c_void_p
_I64 = C.c_int64
_I32 = C.c_int32
_F = C.POINTER(C.c_float)


class BlockDesc(C.Structure):
    _fields_ = [("n", _I64), ("h", _I64), ("w", _I64), ("c0", _I32), ("m", _I32),
                ("k", _I32), ("bk", _I32), ("dtype", _I32), ("layout", _I32)]


class ArenaSizes(C.Structure):
    _fields_ = [(name, _I64) for name in (
        "total_bytes", "feat_offset", "feat_bytes", "z_offset", "z_bytes",
        "stats_offset", "stats_bytes", "acc_offset", "acc_bytes", "g0_offset", "g0_bytes",
        "g1_offset", "g1_bytes", "scratch_offset", "scratch_bytes", "shared1_bytes",
        "shared2_bytes", "param_elems", "stat_elems")]

    def as_dict(self) -> dict:
        return {name: int(getattr(self, name)) for name, _ in self._fields_}


class KernelStat(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("launches", _I64), ("total_ms", C.c_double),
                ("bytes", C.c_double), ("flops", C.c_double), ("bytes_8d", C.c_double)]


class MemoryStats(C.Structure):
    _fields_ = [("live_bytes", _I64 * 6), ("peak_bytes", _I64 * 6), ("total_feature_peak_bytes", _I64),
                ("param_bytes", _I64)]


class ModelDesc(C.Structure):
    _fields_ = [("nblocks", _I32), ("blocks", _I32 * 8), ("k", _I32), ("compression", C.c_double),
                ("classes", _I32), ("c0", _I32), ("in_c", _I32), ("in_h", _I32), ("in_w", _I32),
                ("batch", _I64), ("dtype", _I32), ("stem", _I32)]


# every symbol the header declares: (name, restype, argtypes)
SIGNATURES = {
    "dpb_last_error": (C.c_char_p, []),
    "dpb_version": (C.c_char_p, []),
    "dpb_block_plan": (C.c_int, [C.POINTER(BlockDesc), C.POINTER(ArenaSizes)]),
    "dpb_block_param_elems": (C.c_int, [C.POINTER(BlockDesc), C.POINTER(_I64), C.POINTER(_I64)]),
    "dpb_block_create": (C.c_int, [C.POINTER(BlockDesc), C.c_int, _P, C.POINTER(_P)]),
    "dpb_block_destroy": (C.c_int, [_P]),
    "dpb_block_set_stream": (C.c_int, [_P, _P]),
    "dpb_block_arena": (C.c_int, [_P, C.POINTER(ArenaSizes), C.POINTER(_P)]),
    "dpb_block_forward": (C.c_int, [_P, _P, _P, _P, C.c_int]),
    "dpb_block_forward_eval": (C.c_int, [_P, _P, _P, _P]),
    "dpb_block_backward": (C.c_int, [_P, _P, _P, _P]),
    "dpb_block_read_feats": (C.c_int, [_P, _P]),
    "dpb_block_read_z": (C.c_int, [_P, _P]),
    "dpb_block_read_stats": (C.c_int, [_P, _P]),
    "dpb_sync": (C.c_int, [_P]),
    "dpb_block_launch_count": (_I64, [_P]),
    "dpb_block_profile": (C.c_int, [_P, C.c_int]),
    "dpb_block_profile_read": (C.c_int, [_P, _P, C.c_int, C.POINTER(C.c_int)]),
    "dpb_block_memory": (C.c_int, [C.POINTER(BlockDesc), C.POINTER(_I64), C.POINTER(_I64)]),
    "dpb_selftest_tc_gemm": (C.c_int, [_P, _P, _P, _P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                       C.c_int, _P]),
    "dpb_op_batch_statistics": (C.c_int, [_P, _I64, _I64, _I64, _I64, _P, _P, _P]),
    "dpb_op_batchnorm_apply": (C.c_int, [_P, _I64, _I64, _I64, _I64, _P, _P, _P, _P, C.c_int, _P, _P]),
    "dpb_op_batchnorm_backward": (C.c_int, [_P, _P, _I64, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P, _P]),
    "dpb_op_conv2d_forward": (C.c_int, [_P, _I64, _I64, _I64, _I64, _P, _I64, _I64, _I64, _P, _P]),
    "dpb_op_conv2d_backward": (C.c_int, [_P, _P, _I64, _I64, _I64, _I64, _P, _I64, _I64, _I64, _P, _P, _P]),
    "dpb_count_parameters": (C.c_int, [C.c_int, _P, _I32, _I32, C.c_double, _I32, _I32, _I32, C.POINTER(_I64)]),
    "dpb_predict_peak_elements": (C.c_int, [C.c_int, _P, _I32, _I32, C.c_double, _I32, _I32, _I32, _I64,
                                            _I32, _I32, _I32, _P]),
    "dpb_rng_fill_normal": (C.c_int, [C.c_uint64, _P, _I64]),
    "dpb_op_concat_forward": (C.c_int, [C.c_int, _P, _P, _I64, _I64, _I64, _P, _I64, _P]),
    "dpb_op_concat_backward": (C.c_int, [_P, _I64, _I64, _I64, _I64, C.c_int, _P, _P, _P]),
    "dpb_op_relu_forward": (C.c_int, [_P, _I64, _P, _P]),
    "dpb_op_relu_backward": (C.c_int, [_P, _P, _I64, _P, _P]),
    "dpb_model_sizes": (C.c_int, [C.POINTER(ModelDesc), C.POINTER(_I64), C.POINTER(_I64)]),
    "dpb_model_init_params": (C.c_int, [C.POINTER(ModelDesc), C.c_uint64, _P]),
    "dpb_model_create": (C.c_int, [C.POINTER(ModelDesc), C.c_int, _P, C.POINTER(_P)]),
    "dpb_model_destroy": (None, [_P]),
    "dpb_model_step": (C.c_int, [_P, _P, _P, _P, _P, _P, _P]),
    "dpb_model_sync": (C.c_int, [_P]),
    "dpb_model_wait_input": (C.c_int, [_P, _P]),
    "dpb_model_memory_stats": (C.c_int, [_P, C.POINTER(MemoryStats)]),
    "dpb_model_set_comm": (C.c_int, [_P, _P]),
    "dpb_model_buckets": (C.c_int, [C.POINTER(ModelDesc), _P, C.c_int, C.POINTER(C.c_int)]),
    "dpb_comm_unique_id": (C.c_int, [_P]),
    "dpb_comm_init": (C.c_int, [C.c_int, C.c_int, _P, C.c_int, C.POINTER(_P)]),
    "dpb_comm_destroy": (C.c_int, [_P]),
    "dpb_comm_check": (C.c_int, [_P]),
    "dpb_model_launch_count": (_I64, [_P]),
    "dpb_block_memory_stats": (C.c_int, [_P, C.POINTER(MemoryStats)]),
    "dpb_block_trace": (C.c_int, [_P, _P, C.c_int, _P, C.POINTER(C.c_int)]),
    "dpb_sgd_step": (C.c_int, [_P, _P, _P, _I64, C.c_double, C.c_double, C.c_double, C.c_int, _P]),
    "dpb_lr_at": (C.c_int, [C.c_int, C.c_double, C.c_int, _P, C.c_int, C.c_double, C.c_double, C.c_int,
                            C.POINTER(C.c_double)]),
    "dpb_checkpoint_save": (C.c_int, [C.c_char_p, C.c_int, _P, _P, _P, C.c_int]),
    "dpb_checkpoint_load": (C.c_int, [C.c_char_p, C.c_int, _P, _P, _P, C.POINTER(C.c_int)]),
}

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA extension first "
                "(python -m paper_1707_06990_b200.build); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    """Raise the reference-named exception for a non-zero status."""
    if rc != 0:
        msg = lib().dpb_last_error().decode(errors="replace")
        raise errors.from_status(rc, msg)
