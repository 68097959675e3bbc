"""ctypes binding of libkc.so (include/kclique.h).

There is no fallback: if the shared library is missing or no sm_100 device is
visible, every compute call raises.  ``status`` codes map onto the reference's
exception classes (scheduler.py:188-200 ValueError, :243-244 OverflowError).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libkc.so")

KC_OK, KC_EINVAL, KC_EOVERFLOW, KC_ECUDA, KC_ENOMEM = 0, 1, 3, 4, 5
CRIT = {"degree": 0, "degeneracy": 1, "given": 2, "degeneracy_exact": 3, "degeneracy_bulk": 4}
ALGO = {"orient": 0, "pivot": 1}
SCHEME = {"vertex": 0, "edge": 1}

# every symbol include/kclique.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "kc_abi_version", "kc_last_error", "kc_device_count", "kc_num_sms",
    "kc_normalize_edges", "kc_graph_from_raw_edges", "kc_graph_from_edges", "kc_graph_from_csr", "kc_graph_info", "kc_graph_download",
    "kc_graph_free", "kc_graph_stream", "kc_orient", "kc_dag_download", "kc_count", "kc_num_tasks",
    "kc_task_costs", "kc_shard_ranges", "kc_extract", "kc_count_bitgraph", "kc_find_pivot", "kc_probe",
)


class KcDagInfo(ctypes.Structure):
    _fields_ = [("m_dir", ctypes.c_int64), ("d_max", ctypes.c_int64),
                ("degeneracy", ctypes.c_int64), ("rounds", ctypes.c_int64),
                ("rank_ms", ctypes.c_double), ("orient_ms", ctypes.c_double)]


class KcCountArgs(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int32), ("algorithm", ctypes.c_int32),
                ("scheme", ctypes.c_int32), ("all_k", ctypes.c_int32),
                ("group_size", ctypes.c_int32), ("block_size", ctypes.c_int32),
                ("task_lo", ctypes.c_int64), ("task_hi", ctypes.c_int64)]


class KcCountRaw(ctypes.Structure):
    _fields_ = [("limbs", ctypes.c_uint64 * 4), ("visits", ctypes.c_uint64),
                ("tasks_run", ctypes.c_uint64), ("hist_dim", ctypes.c_int64),
                ("count_ms", ctypes.c_double), ("group_size", ctypes.c_int32),
                ("launches", ctypes.c_int32),
                ("word_ops", ctypes.c_uint64), ("extract_bytes", ctypes.c_uint64)]


class KcError(RuntimeError):
    """A CUDA-side failure (status KC_ECUDA)."""


_lib = None
_P = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def load(path: str = LIB_PATH):
    """Load libkc.so; raises (no fallback) when it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -m paper_2104_13209_b200.build` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(path)
    sig = {
        "kc_abi_version": (ctypes.c_int, []),
        "kc_last_error": (ctypes.c_char_p, []),
        "kc_device_count": (ctypes.c_int, []),
        "kc_num_sms": (ctypes.c_int, [ctypes.c_int]),
        "kc_normalize_edges": (ctypes.c_int, [ctypes.c_int, _P, _i64, _P, ctypes.POINTER(_i64),
                                              _P, ctypes.POINTER(_i64), ctypes.POINTER(_i64),
                                              ctypes.POINTER(_i64),
                                              ctypes.POINTER(ctypes.c_double)]),
        "kc_graph_from_raw_edges": (ctypes.c_int, [ctypes.c_int, _P, _i64, ctypes.POINTER(_i64),
                                                   ctypes.POINTER(_i64),
                                                   ctypes.POINTER(ctypes.c_double),
                                                   ctypes.POINTER(_P)]),
        "kc_graph_from_edges": (ctypes.c_int, [ctypes.c_int, _P, _i64, _P, _i64,
                                               ctypes.POINTER(_P)]),
        "kc_graph_from_csr": (ctypes.c_int, [ctypes.c_int, _i64, _i64, _P, _P, _P,
                                             ctypes.POINTER(_P)]),
        "kc_graph_info": (ctypes.c_int, [_P, ctypes.POINTER(_i64), ctypes.POINTER(_i64),
                                         ctypes.POINTER(_i64), ctypes.POINTER(ctypes.c_double)]),
        "kc_graph_download": (ctypes.c_int, [_P, _P, _P, _P, _P]),
        "kc_graph_free": (None, [_P]),
        "kc_graph_stream": (ctypes.c_int, [_P, ctypes.POINTER(_P)]),
        "kc_orient": (ctypes.c_int, [_P, ctypes.c_int, _P, ctypes.POINTER(KcDagInfo)]),
        "kc_dag_download": (ctypes.c_int, [_P, _P, _P, _P, _P]),
        "kc_count": (ctypes.c_int, [_P, ctypes.POINTER(KcCountArgs), ctypes.POINTER(KcCountRaw),
                                    _P, _i64, _P, _i32]),
        "kc_num_tasks": (ctypes.c_int, [_P, _i32, ctypes.POINTER(_i64)]),
        "kc_task_costs": (ctypes.c_int, [_P, ctypes.POINTER(KcCountArgs), _P, _i64]),
        "kc_shard_ranges": (ctypes.c_int, [_P, ctypes.POINTER(KcCountArgs), _i32, _P]),
        "kc_extract": (ctypes.c_int, [_P, _i32, _i64, _i32, _P, _P, _i64, _i64,
                                      ctypes.POINTER(_i64)]),
        "kc_count_bitgraph": (ctypes.c_int, [ctypes.c_int, _P, _i64, _i32, _i32, _i32, _P, _P,
                                             _P]),
        "kc_probe": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                    ctypes.POINTER(ctypes.c_double),
                                    ctypes.POINTER(ctypes.c_double)]),
        "kc_find_pivot": (ctypes.c_int, [ctypes.c_int, _P, _i64, _P, ctypes.POINTER(_i64), _P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    if L.kc_abi_version() != 2:
        raise ImportError("libkc ABI version mismatch")
    _lib = L
    return L


def check(status: int) -> None:
    if status == KC_OK:
        return
    msg = (load().kc_last_error() or b"").decode(errors="replace")
    if status == KC_EINVAL:
        raise ValueError(msg)
    if status == KC_EOVERFLOW:
        raise OverflowError(msg or "k-clique count exceeded the 128-bit accumulator")
    if status == KC_ENOMEM:
        raise MemoryError(msg)
    raise KcError(msg)


def device_count() -> int:
    return int(load().kc_device_count())


def num_sms(device: int = 0) -> int:
    return int(load().kc_num_sms(device))


def graph_stream(handle) -> int:
    """cudaStream_t (as an int) the library issues this graph's work on."""
    s = ctypes.c_void_p()
    check(load().kc_graph_stream(handle, ctypes.byref(s)))
    return int(s.value or 0)


def current_device() -> int:
    """Device for new graphs: $KC_DEVICE, else LOCAL_RANK (one process per GPU)."""
    for var in ("KC_DEVICE", "LOCAL_RANK"):
        v = os.environ.get(var)
        if v is not None and v.strip() != "":
            return int(v)
    return 0
