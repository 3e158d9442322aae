"""ctypes binding of libkvswap.so (include/kvswap.h).

This is the product path: there is no CPU fallback.  If the shared library
is missing or fails to load, every data-plane call raises NativeLibraryError.
Return codes map onto the reference's exception vocabulary: bad arguments
raise ValueError (as kvswitch does, e.g. alloc.py:233-234), ops outside a pool
raise IndexError, CUDA failures raise KvSwapCudaError.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path
from typing import Optional

LIB_PATH = Path(__file__).resolve().parent / "libkvswap.so"

KVS_OK = 0
KVS_ERR_INVALID = -1
KVS_ERR_RANGE = -2
KVS_ERR_ALIGN = -3
KVS_ERR_NOMEM = -4
KVS_ERR_UNSUPPORTED = -5

KVS_DIR_OUT = 0
KVS_DIR_IN = 1

KVS_BASE_PER_BLOCK = 0
KVS_BASE_PER_RUN = 1
KVS_BASE_BATCH = 2

KVS_PATH_LSU = 0
KVS_PATH_BULK = 1
PATHS = {"lsu": KVS_PATH_LSU, "bulk": KVS_PATH_BULK}

KVS_HOST_DEFAULT = 0
KVS_HOST_REGISTER = 1
KVS_HOST_WRITE_COMBINED = 2

# Every symbol include/kvswap.h declares; tests assert all are exported.
EXPORTED_SYMBOLS = (
    "kvs_abi_version",
    "kvs_error_string",
    "kvs_create",
    "kvs_destroy",
    "kvs_set_launch",
    "kvs_set_path",
    "kvs_set_pace",
    "kvs_set_budget",
    "kvs_set_budget_priority",
    "kvs_set_budget_share",
    "kvs_set_pace_burst",
    "kvs_swap",
    "kvs_swap_layered",
    "kvs_set_layer_group",
    "kvs_swap_ops",
    "kvs_swap_signaled",
    "kvs_wait_flag",
    "kvs_launch_count",
    "kvs_memcpy_baseline",
    "kvs_set_staging",
    "kvs_host_alloc",
    "kvs_host_free",
    "kvs_sm_partition",
    "kvs_stream_read",  # include/kvswap_workload.h
    "kvs_stream_read_ex",  # include/kvswap_workload.h
    "kvs_graph_create", "kvs_graph_destroy", "kvs_graph_stream", "kvs_graph_begin",
    "kvs_graph_mark", "kvs_graph_end", "kvs_graph_launch", "kvs_graph_elapsed",
    "kvs_graph_stats",  # include/kvswap_workload.h
    "kvs_graph_decode_step",  # include/kvswap_workload.h
    "kvs_kv_tokens",  # include/kvswap_workload.h
)

DIRECTIONS = {"out": KVS_DIR_OUT, "in": KVS_DIR_IN}


class NativeLibraryError(RuntimeError):
    """libkvswap.so is missing or unusable; the data plane has no fallback."""


class KvSwapCudaError(RuntimeError):
    """A CUDA runtime/driver call inside libkvswap failed."""


class KvsSignals(ctypes.Structure):
    _fields_ = [
        ("op_flags", ctypes.c_void_p),
        ("plane_flags", ctypes.c_void_p),
        ("done_flag", ctypes.c_void_p),
        ("seq", ctypes.c_uint32),
        ("reserved", ctypes.c_uint32),
    ]


class KvsDecodeStep(ctypes.Structure):
    """include/kvswap_workload.h KvsDecodeStep."""
    _fields_ = [
        ("segs", ctypes.c_void_p),
        ("n_segs", ctypes.c_int32),
        ("block_tokens", ctypes.c_int32),
        ("mismatch", ctypes.c_void_p),
        ("weights", ctypes.c_void_p),
        ("weight_bytes", ctypes.c_uint64),
        ("w_bytes_per_layer", ctypes.c_uint64),
        ("sink", ctypes.c_void_p),
        ("w_ctas", ctypes.c_int32),
        ("n_deps", ctypes.c_int32),
        ("dep_flags", ctypes.c_void_p),
        ("dep_seqs", ctypes.c_void_p),
        ("marks", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


class KvsGeometry(ctypes.Structure):
    _fields_ = [
        ("num_planes", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("plane_chunk_bytes", ctypes.c_int64),
        ("plane_block_stride", ctypes.c_int64),
    ]


_lib: Optional[ctypes.CDLL] = None


def _declare(lib: ctypes.CDLL) -> None:
    c = ctypes
    lib.kvs_abi_version.restype = c.c_int
    lib.kvs_abi_version.argtypes = []
    lib.kvs_error_string.restype = c.c_char_p
    lib.kvs_error_string.argtypes = [c.c_int]
    lib.kvs_create.restype = c.c_int
    lib.kvs_create.argtypes = [
        c.c_int, c.POINTER(KvsGeometry), c.POINTER(c.c_uint64), c.c_void_p,
        c.c_int64, c.c_int64, c.POINTER(c.c_void_p),
    ]
    lib.kvs_destroy.restype = c.c_int
    lib.kvs_destroy.argtypes = [c.c_void_p]
    lib.kvs_set_launch.restype = c.c_int
    lib.kvs_set_launch.argtypes = [c.c_void_p, c.c_int, c.c_int, c.c_int]
    lib.kvs_set_path.restype = c.c_int
    lib.kvs_set_path.argtypes = [c.c_void_p, c.c_int, c.c_int, c.c_int, c.c_int]
    lib.kvs_set_pace.restype = c.c_int
    lib.kvs_set_pace.argtypes = [c.c_void_p, c.c_int, c.c_double]
    lib.kvs_set_budget.restype = c.c_int
    lib.kvs_set_budget.argtypes = [c.c_void_p, c.c_double]
    lib.kvs_set_budget_priority.restype = c.c_int
    lib.kvs_set_budget_priority.argtypes = [c.c_void_p, c.c_int]
    lib.kvs_set_pace_burst.restype = c.c_int
    lib.kvs_set_pace_burst.argtypes = [c.c_void_p, c.c_int, c.c_int64]
    lib.kvs_set_budget_share.restype = c.c_int
    lib.kvs_set_budget_share.argtypes = [c.c_void_p, c.c_int, c.c_double]
    lib.kvs_set_layer_group.restype = c.c_int
    lib.kvs_set_layer_group.argtypes = [c.c_void_p, c.c_int]
    lib.kvs_swap.restype = c.c_int
    lib.kvs_swap.argtypes = [
        c.c_void_p, c.c_int, c.c_void_p, c.c_int32, c.c_uint64, c.c_void_p, c.c_uint32,
    ]
    lib.kvs_swap_layered.restype = c.c_int
    lib.kvs_swap_layered.argtypes = [
        c.c_void_p, c.c_int, c.c_void_p, c.c_int32, c.c_uint64, c.c_void_p, c.c_uint32,
    ]
    lib.kvs_swap_ops.restype = c.c_int
    lib.kvs_swap_ops.argtypes = [
        c.c_void_p, c.c_int, c.c_void_p, c.c_int32, c.c_uint64, c.c_void_p, c.c_void_p,
        c.c_uint32,
    ]
    lib.kvs_swap_signaled.restype = c.c_int
    lib.kvs_swap_signaled.argtypes = [c.c_void_p, c.c_int, c.c_void_p, c.c_int32, c.c_uint64,
                                      c.POINTER(KvsSignals)]
    lib.kvs_wait_flag.restype = c.c_int
    lib.kvs_wait_flag.argtypes = [c.c_uint64, c.c_void_p, c.c_uint32]
    lib.kvs_launch_count.restype = c.c_int64
    lib.kvs_launch_count.argtypes = [c.c_void_p]
    lib.kvs_memcpy_baseline.restype = c.c_int
    lib.kvs_memcpy_baseline.argtypes = [
        c.c_void_p, c.c_int, c.c_int, c.c_void_p, c.c_int32, c.c_uint64,
    ]
    lib.kvs_set_staging.restype = c.c_int
    lib.kvs_set_staging.argtypes = [c.c_void_p, c.c_int64, c.c_int]
    lib.kvs_host_alloc.restype = c.c_int
    lib.kvs_host_alloc.argtypes = [
        c.c_size_t, c.c_int, c.c_int, c.POINTER(c.c_void_p), c.POINTER(c.c_void_p),
    ]
    lib.kvs_host_free.restype = c.c_int
    lib.kvs_host_free.argtypes = [c.c_void_p]
    lib.kvs_sm_partition.restype = c.c_int
    lib.kvs_sm_partition.argtypes = [c.c_int, c.c_int, c.c_int, c.c_int, c.c_int,
                                     c.POINTER(c.c_uint64), c.POINTER(c.c_uint64),
                                     c.POINTER(c.c_int)]
    lib.kvs_stream_read.restype = c.c_int
    lib.kvs_stream_read.argtypes = [c.c_int, c.c_uint64, c.c_void_p, c.c_size_t, c.c_size_t,
                                    c.c_int, c.c_void_p]
    lib.kvs_stream_read_ex.restype = c.c_int
    lib.kvs_stream_read_ex.argtypes = [c.c_int, c.c_uint64, c.c_void_p, c.c_size_t, c.c_size_t,
                                       c.c_int, c.c_void_p, c.c_int]
    lib.kvs_graph_create.restype = c.c_int
    lib.kvs_graph_create.argtypes = [c.c_int, c.c_int, c.POINTER(c.c_void_p)]
    lib.kvs_graph_destroy.restype = c.c_int
    lib.kvs_graph_destroy.argtypes = [c.c_void_p]
    lib.kvs_graph_stream.restype = c.c_int
    lib.kvs_graph_stream.argtypes = [c.c_void_p, c.POINTER(c.c_uint64)]
    lib.kvs_graph_begin.restype = c.c_int
    lib.kvs_graph_begin.argtypes = [c.c_void_p]
    lib.kvs_graph_mark.restype = c.c_int
    lib.kvs_graph_mark.argtypes = [c.c_void_p, c.c_int]
    lib.kvs_graph_end.restype = c.c_int
    lib.kvs_graph_end.argtypes = [c.c_void_p, c.POINTER(c.c_int)]
    lib.kvs_graph_launch.restype = c.c_int
    lib.kvs_graph_launch.argtypes = [c.c_void_p, c.c_uint64]
    lib.kvs_graph_elapsed.restype = c.c_int
    lib.kvs_graph_elapsed.argtypes = [c.c_void_p, c.c_int, c.c_int, c.POINTER(c.c_float)]
    lib.kvs_graph_stats.restype = c.c_int
    lib.kvs_graph_stats.argtypes = [c.c_void_p, c.POINTER(c.c_int64)]
    lib.kvs_graph_decode_step.restype = c.c_int
    lib.kvs_graph_decode_step.argtypes = [c.c_void_p, c.c_void_p, c.POINTER(KvsDecodeStep),
                                          c.POINTER(c.c_int)]
    lib.kvs_kv_tokens.restype = c.c_int
    lib.kvs_kv_tokens.argtypes = [c.c_void_p, c.c_int, c.c_void_p, c.c_int32, c.c_int32,
                                  c.c_int32, c.c_int32, c.c_uint64, c.c_void_p]


def load(path: Optional[os.PathLike] = None) -> ctypes.CDLL:
    """Load (once) and type the native library; raise if it is unusable."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise NativeLibraryError(
            f"{p} not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    try:
        lib = ctypes.CDLL(str(p))
    except OSError as exc:
        raise NativeLibraryError(f"cannot load {p}: {exc}") from exc
    missing = [s for s in EXPORTED_SYMBOLS if not hasattr(lib, s)]
    if missing:
        raise NativeLibraryError(f"{p} lacks symbols {missing}")
    _declare(lib)
    if lib.kvs_abi_version() != 1:
        raise NativeLibraryError(f"{p}: ABI {lib.kvs_abi_version()} != 1")
    if path is None:
        _lib = lib
    return lib


def error_string(code: int) -> str:
    return load().kvs_error_string(int(code)).decode()


def check(code: int, what: str = "kvswap") -> None:
    """Map a libkvswap return code onto the reference's exception types."""
    if code == KVS_OK:
        return
    msg = f"{what}: {error_string(code)} (code {code})"
    if code in (KVS_ERR_INVALID, KVS_ERR_ALIGN):
        raise ValueError(msg)
    if code == KVS_ERR_RANGE:
        raise IndexError(msg)
    if code == KVS_ERR_NOMEM:
        raise MemoryError(msg)
    raise KvSwapCudaError(msg)
