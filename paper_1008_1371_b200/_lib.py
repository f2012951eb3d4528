"""ctypes binding of libhsvd_b200.so (the C ABI declared in
include/hsvd_b200.h).  There is no fallback: if the library is missing or no
CUDA device is present, every compute entry point raises."""

import ctypes
import os

from .errors import (DefinitenessLostError, HsvdCudaError, NumericalSingularityError,
                     RankDeficiencyError,
                     ShapeError)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libhsvd_b200.so")

HSVD_OK = 0
HSVD_DEFINITENESS_LOST = 1
HSVD_RANK_DEFICIENT = 2
HSVD_SHAPE_ERROR = 3
HSVD_NUMERICAL_SINGULARITY = 4
HSVD_ERR_CUDA = -1
HSVD_ERR_ARG = -2
HSVD_ERR_UNSUPPORTED = -3

MODE_POINTWISE = 0
MODE_BLOCK = 1
SCHEDULE_MODULUS = 0
SCHEDULE_ROW_CYCLIC = 1

#: every symbol include/hsvd_b200.h declares (checked by the CPU tests)
EXPORTED = (
    "hsvd_last_error", "hsvd_version", "hsvd_abi_sizes", "hsvd_default_config",
    "hsvd_dot_chunked", "hsvd_fused_pair_update", "hsvd_rotation_batch",
    "hsvd_precompute", "hsvd_step_blocks", "hsvd_advance_stepper",
    "hsvd_stepper_init", "hsvd_sort_diagonal", "hsvd_reduce_sweep",
    "hsvd_extract", "hsvd_drive_workspace_size", "hsvd_drive",
    "hsvd_drive_host",
    "hsvd_comm_unique_id", "hsvd_comm_init", "hsvd_comm_destroy",
    "hsvd_shard_columns", "hsvd_sharded_workspace_size", "hsvd_drive_sharded",
    "hsvd_plan_create", "hsvd_plan_destroy", "hsvd_plan_advance", "hsvd_plan_state",
    "hsvd_plan_redistribute", "hsvd_plan_place",
    "hsvd_bp_workspace_size", "hsvd_bp_factor", "hsvd_bp_factor_dd", "hsvd_qr_workspace_size",
    "hsvd_qr_shorten", "hsvd_gen_workspace_size", "hsvd_gen_init", "hsvd_gen_reflect",
    "hsvd_gen_finish",
)


class HsvdConfigC(ctypes.Structure):
    _fields_ = [
        ("max_sweeps", ctypes.c_int64),
        ("eps", ctypes.c_double),
        ("teps", ctypes.c_double),
        ("accumulate_v", ctypes.c_int32),
        ("use_skip", ctypes.c_int32),
        ("chunk", ctypes.c_int64),
        ("schedule", ctypes.c_int32),
        ("sort", ctypes.c_int32),
        ("mode", ctypes.c_int32),
        ("block_cols", ctypes.c_int32),
        ("inner_full", ctypes.c_int32),
        ("use_graph", ctypes.c_int32),
        ("profile", ctypes.c_int32),
        ("block_rotation", ctypes.c_int32),
        ("inner_passes", ctypes.c_int32),
        ("block_streams", ctypes.c_int32),
    ]


class HsvdResultC(ctypes.Structure):
    _fields_ = [
        ("sweeps_used", ctypes.c_int64),
        ("stop_reason", ctypes.c_int32),
        ("status", ctypes.c_int32),
        ("rotations", ctypes.c_int64),
        ("skips", ctypes.c_int64),
        ("err", ctypes.c_int64 * 3),
        ("launches", ctypes.c_int64),
        ("setup_ms", ctypes.c_double),
        ("sweeps_ms", ctypes.c_double),
        ("finish_ms", ctypes.c_double),
        ("kernel_ms", ctypes.c_double * 4),
        ("kernel_launches", ctypes.c_int64 * 4),
    ]


class HsvdTelemetryC(ctypes.Structure):
    _fields_ = [
        ("sweep", ctypes.c_int64),
        ("rotations", ctypes.c_int64),
        ("skips", ctypes.c_int64),
        ("max_t", ctypes.c_double),
        ("gpu_ms", ctypes.c_double),
    ]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_D = ctypes.c_double

_SIGS = {
    "hsvd_last_error": (ctypes.c_char_p, []),
    "hsvd_version": (ctypes.c_int, []),
    "hsvd_abi_sizes": (None, [_P]),
    "hsvd_default_config": (None, [ctypes.POINTER(HsvdConfigC)]),
    "hsvd_dot_chunked": (ctypes.c_int, [_P, _P, _I64, _I64, _P, _P]),
    "hsvd_fused_pair_update": (ctypes.c_int, [_P, _P, _I64, _D, _D, _D, _P]),
    "hsvd_rotation_batch": (ctypes.c_int, [_P, _P, _P, _P, _I64, _P, _P, _P, _P]),
    "hsvd_precompute": (ctypes.c_int, [_P, _I64, _I64, _I64, _I64, _P, _P, _P]),
    "hsvd_step_blocks": (ctypes.c_int, [_P, _I64, _I64, _P, _I64, _I64, _P, _P,
                                        _P, _P, _P, _P, _P, _I64, _P, _I64,
                                        _I64, _D, _D, _I32, _I64, _I32, _P, _P,
                                        _P, _P, _P]),
    "hsvd_advance_stepper": (ctypes.c_int, [_P, _P, _P, _P, _I64, _I64, _P]),
    "hsvd_stepper_init": (ctypes.c_int, [_P, _P, _P, _P, _I64, _P]),
    "hsvd_sort_diagonal": (ctypes.c_int, [_P, _P, _P, _I64, _I64, _P, _P]),
    "hsvd_reduce_sweep": (ctypes.c_int, [_P, _I64, _P, _P, _P, _I64, _P, _I32, _P]),
    "hsvd_extract": (ctypes.c_int, [_P, _I64, _I64, _P, _P, _P, _I64, _P, _P, _P]),
    "hsvd_drive_workspace_size": (ctypes.c_int64, [_I64, _I64, ctypes.POINTER(HsvdConfigC)]),
    "hsvd_drive": (ctypes.c_int, [_P, _I64, _I64, _I64, _P, _I64, _P, _I64,
                                  ctypes.POINTER(HsvdConfigC), _P, _P, _P, _I64,
                                  ctypes.POINTER(HsvdResultC),
                                  ctypes.POINTER(HsvdTelemetryC), _P]),
    "hsvd_drive_host": (ctypes.c_int, [_P, _I64, _I64, _P, _I64,
                                       ctypes.POINTER(HsvdConfigC), _P, _P, _P,
                                       _P, ctypes.POINTER(HsvdResultC),
                                       ctypes.POINTER(HsvdTelemetryC)]),
    "hsvd_comm_unique_id": (ctypes.c_int, [_P]),
    "hsvd_comm_init": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_P)]),
    "hsvd_comm_destroy": (ctypes.c_int, [_P]),
    "hsvd_shard_columns": (ctypes.c_int64, [_I64, _I32, _I32, _I32]),
    "hsvd_sharded_workspace_size": (ctypes.c_int64, [_I64, _I64, _I32, _I32,
                                                     ctypes.POINTER(HsvdConfigC)]),
    "hsvd_drive_sharded": (ctypes.c_int, [_P, _I32, _I32, _P, _P, _P, _I64, _I64, _I64, _P,
                                          _I64, ctypes.POINTER(HsvdConfigC), _P, _P, _P, _P,
                                          _P, _P, _P, ctypes.POINTER(HsvdResultC),
                                          ctypes.POINTER(HsvdTelemetryC)]),
    "hsvd_plan_create": (_P, [_I64, _I32]),
    "hsvd_plan_destroy": (None, [_P]),
    "hsvd_plan_advance": (ctypes.c_int64, [_P, _P, _I64]),
    "hsvd_plan_state": (ctypes.c_int, [_P, _P, _P, _P, _P, _P]),
    "hsvd_plan_redistribute": (ctypes.c_int, [_P, _I32, _P, _P, _I64, _I32, _P, _P, _P, _P]),
    "hsvd_plan_place": (None, [_P]),
    "hsvd_bp_workspace_size": (ctypes.c_int, [_I64, _P]),
    "hsvd_bp_factor": (ctypes.c_int, [_P, _I64, _I64, _D, _P, _I64, _P, _P, _P, _P, _P,
                                      ctypes.c_size_t, _P]),
    "hsvd_bp_factor_dd": (ctypes.c_int, [_P, _P, _I64, _I64, _D, _P, _I64, _P, _P, _P, _P, _P,
                                         ctypes.c_size_t, _P]),
    "hsvd_gen_workspace_size": (ctypes.c_int, [_I64, _P]),
    "hsvd_gen_init": (ctypes.c_int, [_P, _I64, _P, _P, _P]),
    "hsvd_gen_reflect": (ctypes.c_int, [_P, _P, _I64, _P, _I64, _P, ctypes.c_size_t, _P]),
    "hsvd_gen_finish": (ctypes.c_int, [_P, _P, _I64, _P]),
    "hsvd_qr_workspace_size": (ctypes.c_int, [_I64, _I64, _P]),
    "hsvd_qr_shorten": (ctypes.c_int, [_P, _I64, _I64, _I64, _P, _I64, _P, _I64, _P, _P,
                                       ctypes.c_size_t, _P]),
}

_lib = None


def load():
    """Load the in-tree library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; "
                "g.build()'` (there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error():
    return load().hsvd_last_error().decode(errors="replace")


def check(status, err=None):
    """Map a C status to the reference's exception types (errors.py:4-30)."""
    if status == HSVD_OK:
        return
    msg = last_error()
    if status == HSVD_DEFINITENESS_LOST:
        e = tuple(err) if err is not None else (-1, -1, -1)
        raise DefinitenessLostError(int(e[0]), int(e[1]), int(e[2]))
    if status == HSVD_RANK_DEFICIENT:
        raise RankDeficiencyError(msg)
    if status == HSVD_SHAPE_ERROR:
        raise ShapeError(msg)
    if status == HSVD_NUMERICAL_SINGULARITY:
        raise NumericalSingularityError(msg)
    if status == HSVD_ERR_ARG:
        raise ValueError(msg)
    if status == HSVD_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise HsvdCudaError(msg)
