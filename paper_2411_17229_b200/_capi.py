"""ctypes binding of libdade_gpu.so (the C ABI declared in include/dade_gpu.h).

The product path has no CPU fallback: if the shared library (built by
``__graft_entry__.build()`` / ``paper_2411_17229_b200/build.py``) is missing or
fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libdade_gpu.so"


class DadeError(RuntimeError):
    """Base class of the errors the C ABI reports."""


class ConfigError(DadeError):
    """dade::ConfigError — inconsistent parameters or mismatched artifacts
    (proj/include/dade/error.hpp:10-13)."""


class InvalidInput(DadeError, ValueError):
    """dade::InvalidInput — an operation precondition is violated
    (proj/include/dade/error.hpp:15-19)."""


class CudaError(DadeError):
    """A CUDA runtime or launch failure."""


_ERRORS = {1: DadeError, 2: ConfigError, 3: InvalidInput, 4: CudaError}

# flags
QUERIES_RAW = 1
DEVICE_PTRS = 2
MEASURE_FAILURES = 4
# strategy kinds
FD, ADS, DADE = 0, 1, 2


class Stats(C.Structure):
    _fields_ = [("total_dco", C.c_uint64), ("dims_accumulated", C.c_uint64),
                ("eligible", C.c_uint64), ("failures", C.c_uint64)]


def _load():
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA extension first (python __graft_entry__.py build)")
    lib = C.CDLL(str(LIB_PATH))
    P, U32, U64, I, D = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int, C.c_double
    sigs = {
        "dade_gpu_last_error": ([], C.c_char_p),
        "dade_gpu_version": ([], C.c_char_p),
        "dade_gpu_create": ([I, C.POINTER(P)], I),
        "dade_gpu_destroy": ([P], I),
        "dade_gpu_set_stream": ([P, P], I),
        "dade_gpu_synchronize": ([P], I),
        "dade_gpu_set_transform": ([P, U32, P, P], I),
        "dade_gpu_set_ivf": ([P, U32, U32, U32, U32, U32, P, P, P, P], I),
        "dade_gpu_set_ivf_shard": ([P, P], I),
        "dade_gpu_set_base": ([P, U32, U32, P, U32], I),
        "dade_gpu_set_strategy": ([P, U32, U32, U32, P, P, P], I),
        "dade_gpu_set_strategy_dade": ([P, U32, U32, U32, P, P], I),
        "dade_gpu_set_strategy_ads": ([P, U32, U32, D], I),
        "dade_gpu_rotate": ([P, P, U32, P, U32], I),
        "dade_gpu_ivf_search": ([P, P, U32, U32, U32, U32, P, P, P, P], I),
        "dade_gpu_ivf_search_batches": ([P, U32, P, U32, U32, U32, U32, P, P, P, P], I),
        "dade_gpu_flat_search": ([P, P, U32, U32, U32, P, P, P, P], I),
        "dade_gpu_ivf_search_keys": ([P, P, U32, U32, U32, U32, P, P], I),
        "dade_gpu_ivf_search_keys_begin": ([P, P, U32, U32, U32, U32, P, P, P], I),
        "dade_gpu_coarse_probes": ([P, P, U32, U32, U32, P, P], I),
        "dade_gpu_flat_search_keys_begin": ([P, P, U32, U32, U32, P, P], I),
        "dade_gpu_set_seed_rows": ([P, U32], I),
        "dade_gpu_set_graphs": ([P, I], I),
        "dade_gpu_flat_partition": ([P, U32, U32, U64], I),
        "dade_gpu_ivf_search_keys_end": ([P, P, P], I),
        "dade_gpu_flat_search_keys": ([P, P, U32, U32, U32, P, P], I),
        "dade_gpu_merge_keys": ([P, P, U32, U32, U32, P, P, P], I),
        "dade_gpu_dco_evaluate": ([P, P, P, P, U32, U32, P, P, P, P, P], I),
        "dade_gpu_partial_sums": ([P, P, P, U32, U32, P], I),
        "dade_gpu_calibrate": ([P, P, U32, D, U32, U64, U64, U32, P, P, P], I),
        "dade_gpu_launch_count": ([P], U64),
        "dade_gpu_debug_counters": ([P, P], I),
        "dade_gpu_debug_radius": ([P, P, U32], I),
        "dade_gpu_set_profiling": ([P, I], I),
        "dade_gpu_last_scan_profile": ([P, P, P, P], I),
        "dade_gpu_last_filter_profile": ([P, P, P], I),
        "dade_gpu_last_seed_profile": ([P, P, P], I),
        "dade_gpu_set_estimate_dump": ([P, U32], I),
        "dade_gpu_last_union_profile": ([P, P, P], I),
        "dade_gpu_get_stream": ([P, P], I),
        "dade_gpu_index_dims": ([P, P, P], I),
        "dade_gpu_nccl_unique_id": ([P], I),
        "dade_gpu_comm_create": ([P, I, I, P, C.POINTER(P)], I),
        "dade_gpu_comm_destroy": ([P], I),
        "dade_gpu_sharded_ivf_search": ([P, P, U32, U32, U32, U32, P, P, P, P], I),
        "dade_gpu_sharded_flat_search": ([P, P, U32, U32, U32, P, P, P, P], I),
        "dade_gpu_covariance": ([P, P, U32, U32, U32, P, P], I),
        "dade_gpu_kmeans": ([P, P, U32, U32, U32, U32, U64, U32, P, P, P], I),
        "dade_gpu_ivf_build": ([P, P, U32, U32, U32, U32, U64, U32, P, P, P, P], I),
        "dade_gpu_ground_truth": ([P, P, U32, P, U32, U32, U32, U32, P], I),
        "dade_gpu_get_estimate_dump": ([P, U32, P, P, P, P, P, P], I),
    }
    for name, (args, res) in sigs.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


lib = _load()

EXPORTED = [
    "dade_gpu_last_error", "dade_gpu_version", "dade_gpu_create", "dade_gpu_destroy",
    "dade_gpu_set_stream", "dade_gpu_synchronize", "dade_gpu_set_transform", "dade_gpu_set_ivf",
    "dade_gpu_set_ivf_shard", "dade_gpu_set_base", "dade_gpu_set_strategy",
    "dade_gpu_set_strategy_dade", "dade_gpu_set_strategy_ads", "dade_gpu_rotate",
    "dade_gpu_ivf_search", "dade_gpu_ivf_search_batches", "dade_gpu_flat_search", "dade_gpu_ivf_search_keys",
    "dade_gpu_ivf_search_keys_begin", "dade_gpu_ivf_search_keys_end", "dade_gpu_coarse_probes",
    "dade_gpu_flat_search_keys_begin", "dade_gpu_set_seed_rows", "dade_gpu_set_graphs", "dade_gpu_flat_partition",
    "dade_gpu_flat_search_keys", "dade_gpu_merge_keys", "dade_gpu_dco_evaluate",
    "dade_gpu_partial_sums", "dade_gpu_calibrate", "dade_gpu_launch_count",
    "dade_gpu_set_profiling", "dade_gpu_last_scan_profile", "dade_gpu_debug_counters",
    "dade_gpu_last_filter_profile", "dade_gpu_last_seed_profile", "dade_gpu_debug_radius",
    "dade_gpu_set_estimate_dump", "dade_gpu_get_estimate_dump", "dade_gpu_covariance", "dade_gpu_kmeans",
    "dade_gpu_ivf_build", "dade_gpu_ground_truth", "dade_gpu_last_union_profile", "dade_gpu_get_stream",
    "dade_gpu_index_dims", "dade_gpu_nccl_unique_id", "dade_gpu_comm_create", "dade_gpu_comm_destroy",
    "dade_gpu_sharded_ivf_search", "dade_gpu_sharded_flat_search",
]


def check(rc: int) -> None:
    if rc != 0:
        msg = lib.dade_gpu_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, DadeError)(msg)


def ptr(a) -> C.c_void_p:
    """Raw pointer of a numpy array (host) or a torch tensor (device or host)."""
    if a is None:
        return C.c_void_p(None)
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    return C.c_void_p(a.ctypes.data)
