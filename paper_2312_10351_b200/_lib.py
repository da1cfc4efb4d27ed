"""ctypes binding of libopara.so (the C ABI in include/opara.h).

The library is built in-tree (``python -m paper_2312_10351_b200.build``) and
loaded from next to this file.  There is no Python fallback: if the shared
object is missing the import of any hot-path entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from . import errors

_LIB_PATH = Path(__file__).with_name("libopara.so")

OK = 0
_STATUS_TO_EXC = {
    1: errors.FormatError,
    2: errors.GraphValidationError,
    3: errors.PlanViolationError,
    4: errors.CoverageError,
    5: errors.InfeasibleBlockError,
    6: errors.CudaError,
    7: errors.SchedulerError,
    8: ValueError,
    9: KeyError,
    10: errors.SchedulerError,
}


class OparaNode(C.Structure):
    _fields_ = [("id", C.c_int64), ("op_class", C.c_int32), ("_pad", C.c_int32),
                ("num_blocks", C.c_int64), ("threads_per_block", C.c_int64),
                ("shared_mem_per_block", C.c_int64), ("registers_per_thread", C.c_int64)]


NODE_DTYPE = np.dtype([("id", "<i8"), ("op_class", "<i4"), ("_pad", "<i4"),
                       ("num_blocks", "<i8"), ("threads_per_block", "<i8"),
                       ("shared_mem_per_block", "<i8"), ("registers_per_thread", "<i8")])
assert NODE_DTYPE.itemsize == C.sizeof(OparaNode)


class OparaGpuConfig(C.Structure):
    _fields_ = [("num_sms", C.c_int64), ("threads_per_sm", C.c_int64),
                ("shared_mem_per_sm", C.c_int64), ("registers_per_sm", C.c_int64),
                ("max_blocks_per_sm", C.c_int64), ("same_class_slowdown", C.c_double)]


MAX_INTS = 40
MAX_PTRS = 8


class OparaOp(C.Structure):
    _fields_ = [("kind", C.c_int32), ("variant", C.c_int32), ("i", C.c_int64 * MAX_INTS),
                ("f", C.c_double * 4), ("p", C.c_void_p * MAX_PTRS)]


class OparaOpProfile(C.Structure):
    _fields_ = [("num_blocks", C.c_int64), ("threads_per_block", C.c_int64),
                ("shared_mem_per_block", C.c_int64), ("registers_per_thread", C.c_int64),
                ("isolated_us", C.c_double), ("tmem_columns", C.c_int64), ("cluster_size", C.c_int64)]


class OparaSimResult(C.Structure):
    _fields_ = [("makespan_ns", C.c_int64), ("blocked_ns", C.c_int64), ("sync_wait_ns", C.c_int64),
                ("sm_efficiency", C.c_double)]


# Every symbol include/opara.h declares, with its ctypes signature.
_P = C.c_void_p
_I64P = C.POINTER(C.c_int64)
_I32P = C.POINTER(C.c_int32)
SIGNATURES = {
    "opara_last_error": (C.c_char_p, []),
    "opara_version": (C.c_char_p, []),
    "opara_dag_create": (C.c_int, [_P, C.c_int64, _P, C.c_int64, C.POINTER(_P)]),
    "opara_dag_destroy": (None, [_P]),
    "opara_dag_num_nodes": (C.c_int64, [_P]),
    "opara_dag_num_edges": (C.c_int64, [_P]),
    "opara_dag_node_ids": (C.c_int, [_P, _P]),
    "opara_dag_edges": (C.c_int, [_P, _P]),
    "opara_dag_topo_sort": (C.c_int, [_P, _P]),
    "opara_dag_predecessors": (C.c_int, [_P, C.c_int64, _P, C.c_int64, _I64P]),
    "opara_dag_successors": (C.c_int, [_P, C.c_int64, _P, C.c_int64, _I64P]),
    "opara_allocate_streams": (C.c_int, [_P, _P, _I32P, _P, _I64P]),
    "opara_single_stream_plan": (C.c_int, [_P, _P, _I32P]),
    "opara_validate_plan": (C.c_int, [_P, _P, _P, C.c_int64, C.c_int64, _P, C.c_int64,
                                      C.c_char_p, C.c_int64, _I64P]),
    "opara_dominant_share": (C.c_int, [C.POINTER(OparaNode), C.POINTER(OparaGpuConfig),
                                       C.POINTER(C.c_double)]),
    "opara_order": (C.c_int, [_P, C.c_int32, C.POINTER(OparaGpuConfig), _P]),
    "opara_linear_extensions": (C.c_int, [_P, C.c_int64, C.c_int64, _P, _P, _P]),
    "opara_simulate": (C.c_int, [_P, _P, _P, C.c_int32, _P, _P, C.c_int64, C.POINTER(OparaGpuConfig),
                                 C.POINTER(OparaSimResult), _P, _P, _P, _P, C.c_int64, _I64P]),
    "opara_exec_create": (C.c_int, [C.c_int32, _P, C.c_int64, C.POINTER(_P)]),
    "opara_exec_destroy": (None, [_P]),
    "opara_exec_capture": (C.c_int, [_P, C.c_int32, _P, C.c_int32, _P, _P, C.c_int64]),
    "opara_exec_set_priorities": (C.c_int, [_P, _P]),
    "opara_exec_replay": (C.c_int, [_P, C.c_int32, _P]),
    "opara_exec_run_eager": (C.c_int, [_P, _P, C.c_int64, _P]),
    "opara_exec_profile": (C.c_int, [_P, C.c_int32, _P]),
    "opara_exec_trace": (C.c_int, [_P, C.c_int32, _P, _P, _P]),
    "opara_exec_time": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, _P, _P, C.c_int64, _P]),
    "opara_exec_num_launches": (C.c_int64, [_P, C.c_int32]),
    "opara_device_gpu_config": (C.c_int, [C.c_int32, C.POINTER(OparaGpuConfig)]),
    "opara_op_launch_config": (C.c_int, [C.POINTER(OparaOp), C.POINTER(OparaOpProfile)]),
}

_lib = None


def lib() -> C.CDLL:
    """Load libopara.so once; raise loudly if it has not been built."""
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise ImportError(
                f"{_LIB_PATH} is missing: build it with `python -m paper_2312_10351_b200.build` "
                "(there is no Python fallback for the scheduler or the executor)")
        handle = C.CDLL(str(_LIB_PATH), mode=os.RTLD_NOW | getattr(os, "RTLD_GLOBAL", 0))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
        _check_fresh(handle)
    return _lib


def version() -> str:
    return lib().opara_version().decode()


def _check_fresh(handle) -> None:
    """Refuse a libopara.so built from other sources than the ones next to it
    (opara_version() carries the build's source hash, build.source_hash())."""
    if os.environ.get("OPARA_ALLOW_STALE") == "1":
        return
    from . import build
    if not build.CSRC.is_dir():
        return
    got = handle.opara_version().decode().rpartition("src:")[2]
    want = build.source_hash()
    if got != want:
        raise ImportError(f"{_LIB_PATH} is stale: built from sources {got}, the tree has {want}; "
                          "rebuild with `python -m paper_2312_10351_b200.build`")


def check(status: int) -> None:
    """Turn a non-zero opara_status into the reference's exception class."""
    if status == OK:
        return
    msg = lib().opara_last_error().decode("utf-8", "replace")
    exc = _STATUS_TO_EXC.get(status, errors.SchedulerError)
    raise exc(msg)


def ptr(a: np.ndarray) -> int:
    """Address of a contiguous numpy array (None for empty arrays)."""
    if a.size == 0:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def gpu_config_struct(cfg) -> OparaGpuConfig:
    return OparaGpuConfig(int(cfg.num_sms), int(cfg.threads_per_sm), int(cfg.shared_mem_per_sm),
                          int(cfg.registers_per_sm), int(cfg.max_blocks_per_sm),
                          float(getattr(cfg, "same_class_slowdown", 1.4)))
