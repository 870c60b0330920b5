"""ctypes declarations of include/tiletensor_b200.h and the library loader.

The loader fails loudly: if ``_lib/libtiletensor_b200.so`` is missing it raises
(there is no pure-Python or CPU implementation to fall back to).  Run
``python -m paper_2011_01805_b200.build`` or ``__graft_entry__.build()``.
"""
from __future__ import annotations

import ctypes
from pathlib import Path

TT_MAX_RANK = 16  # include/tiletensor_b200.h
LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libtiletensor_b200.so"


class CDim(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("d", ctypes.c_int64), ("t", ctypes.c_int64),
                ("unknown", ctypes.c_int32), ("interleaved", ctypes.c_int32)]


class CShape(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("relaxed", ctypes.c_int32),
                ("dims", CDim * TT_MAX_RANK)]


class CCost(ctypes.Structure):
    _fields_ = [("additions", ctypes.c_uint64), ("multiplications", ctypes.c_uint64),
                ("mask_multiplications", ctypes.c_uint64), ("rotations", ctypes.c_uint64),
                ("bootstraps", ctypes.c_uint64), ("power_of_two_rotations", ctypes.c_uint64)]


_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
_U64 = ctypes.c_uint64
_SP = ctypes.POINTER(CShape)
_I64P = ctypes.POINTER(ctypes.c_int64)

# name: (restype, argtypes)
SIGNATURES = {
    "tt_last_error": (ctypes.c_char_p, []),
    "tt_last_error_position": (_I64, []),
    "tt_version": (ctypes.c_char_p, []),
    "tt_shape_parse": (_I, [ctypes.c_char_p, _SP]),
    "tt_shape_format": (_I, [_SP, ctypes.c_char_p, _I64]),
    "tt_shape_check": (_I, [_SP]),
    "tt_shape_external": (_I, [_SP, _I64P]),
    "tt_shape_tile_count": (_I64, [_SP]),
    "tt_shape_tile_slots": (_I64, [_SP]),
    "tt_shape_used_slots": (_I64, [_SP]),
    "tt_shape_elementwise_result": (_I, [_SP, _SP, _I, _SP]),
    "tt_shape_sum_result": (_I, [_SP, _I, _SP]),
    "tt_logical_indices": (_I, [_SP, _I64P, _I64, _I64P]),
    "tt_slot_of": (_I, [_SP, _I64P, _I64P, _I64P]),
    "tt_rotations_left_to_right": (_I64, [_I64]),
    "tt_rotations_right_to_left": (_I64, [_I64]),
    "tt_device_count": (_I, [ctypes.POINTER(ctypes.c_int)]),
    "tt_session_create": (_I, [_I64, _I64, _I, ctypes.POINTER(_P)]),
    "tt_session_destroy": (None, [_P]),
    "tt_session_slot_count": (_I64, [_P]),
    "tt_session_max_chain_index": (_I64, [_P]),
    "tt_session_device": (_I, [_P]),
    "tt_session_set_stream": (_I, [_P, _P]),
    "tt_session_use_own_stream": (_I, [_P]),
    "tt_session_stream": (_P, [_P]),
    "tt_session_synchronize": (_I, [_P]),
    "tt_session_cost": (None, [_P, ctypes.POINTER(CCost)]),
    "tt_session_reset_counters": (None, [_P]),
    "tt_session_launches": (_U64, [_P]),
    "tt_session_count_bootstraps": (None, [_P, _I64]),
    "tt_device_alloc": (_I, [_P, _I64, ctypes.POINTER(_P)]),
    "tt_device_free": (_I, [_P, _P]),
    "tt_tiles_alloc": (_I, [_P, _I64, ctypes.POINTER(_P)]),
    "tt_tiles_release": (_I, [_P, _P]),
    "tt_copy_h2d": (_I, [_P, _P, _P, _I64]),
    "tt_copy_d2h": (_I, [_P, _P, _P, _I64]),
    "tt_copy_d2d": (_I, [_P, _P, _P, _I64]),
    "tt_fill_uniform": (_I, [_P, _P, _I64, _U64, _I64, ctypes.c_double, ctypes.c_double]),
    "tt_pack": (_I, [_P, _P, _SP, _P]),
    "tt_unpack": (_I, [_P, _SP, _P, _P]),
    "tt_elementwise": (_I, [_P, _I, _SP, _P, _I64, _SP, _P, _I64, _SP, _P, _I64P]),
    "tt_sum": (_I, [_P, _SP, _P, _I, _I, _SP, _P]),
    "tt_mul_sum": (_I, [_P, _SP, _P, _I64, _SP, _P, _I64, _I, _I, _SP, _P, _I64P]),
    "tt_linalg_product": (_I, [_P, _I, _SP, _P, _I64, _SP, _P, _I64, _I, _SP, _P, _I64P]),
    "tt_linalg_chain2": (_I, [_P, _I, _SP, _P, _I64, _SP, _P, _I64, _I, _SP, _P, _I64, _I, _I,
                              _SP, _P, _I64P, _SP, _P, _I64P]),
    "tt_mul_sum_clean": (_I, [_P, _SP, _P, _I64, _SP, _P, _I64, _I, _I, _SP, _P, _I64P]),
    "tt_mul_sum_affine": (_I, [_P, _SP, _P, _I64, _SP, _P, _I64, _I, _I, _SP, _P, _I64, _I, _SP, _P,
                               _I64P]),
    "tt_clean_unknowns": (_I, [_P, _SP, _P, _I64, _SP, _P, _I64P]),
    "tt_replicate_dim": (_I, [_P, _SP, _P, _I, _SP, _P]),
    "tt_tiles_binary": (_I, [_P, _I, _P, _P, _P, _I64, _I64P, _I64P, _I64P]),
    "tt_batch_affine": (_I, [_P, _P, _I64, _I64, _P, _P, _P, _P, _P, _I64, _I64P]),
    "tt_affine_layer_create": (_I, [_P, _I64, _I64, _P, _P, _P, _P, _P]),
    "tt_affine_layer_apply": (_I, [_P, _P, _P, _P, _I64, _I64P]),
    "tt_affine_layer_destroy": (None, [_P, _P]),
    "tt_mul_fold": (_I, [_P, _P, _P, _I64, _P, _P, _I64, _I, _I64, _I64, _P, _P, _I64P]),
    "tt_fold_shape": (_I, [_P, _P, _I, _P]),
    "tt_tiles_mask_mul": (_I, [_P, _P, _P, _P, _I64, _I64P, _I64P]),
    "tt_tiles_rotate": (_I, [_P, _P, _I64, _P, _I64]),
    "tt_sum_tile_strided": (_I, [_P, _P, _I64, _I64, _I, _P, _I64]),
    "tt_sum_tile_dim": (_I, [_P, _P, _I64P, _I, _I, _I, _P, _I64]),
    "tt_replicate_tile_dim": (_I, [_P, _P, _I64P, _I, _I, _P, _I64]),
    "tt_set_kernel_path": (_I, [_I]),
    "tt_kernel_path": (_I, []),
    "tt_set_chain_kernel": (_I, [_I]),
    "tt_chain_kernel": (_I, []),
    "tt_shard_plan": (_I, [_SP, _I, _I, _I, _I64P, _I64P, _SP]),
}

_LIB = None


def lib() -> ctypes.CDLL:
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"native library {LIB_PATH} is missing: build it with "
                "`python -m paper_2011_01805_b200.build` (there is no CPU fallback)")
        handle = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = handle
    return _LIB
