"""ORACLE — ctypes wrapper of oracle/liboracle.so (the C restatement).

Test/bench infrastructure only: used by tests/ to cross-check the numpy
restatement and by bench.py as the timed CPU baseline (`cpu_baseline`,
`--impl reference`).  Never imported by the product package.
"""

from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np

LIB = Path(__file__).resolve().parent / "liboracle.so"
_lib = None


def load() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not LIB.exists():
            import sys
            sys.path.insert(0, str(LIB.parent.parent))
            from paper_2411_18424_b200._build import build_oracle
            build_oracle()
        lib = ctypes.CDLL(str(LIB))
        lib.oracle_apply_plan.restype = ctypes.c_int
        lib.oracle_apply_plan.argtypes = [
            ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int,
        ]
        _lib = lib
    return _lib


def apply_plan(direction: str, plane_ptrs, num_planes: int, chunk: int, stride: int,
               host_ptr: int, ops: np.ndarray, nthreads: int = 1) -> None:
    ops32 = np.ascontiguousarray(ops, dtype=np.int32).reshape(-1, 3)
    ptrs = (ctypes.c_uint64 * num_planes)(*plane_ptrs)
    rc = load().oracle_apply_plan(0 if direction == "out" else 1, ptrs, num_planes, chunk, stride,
                                  ctypes.c_void_p(host_ptr),
                                  ops32.ctypes.data_as(ctypes.c_void_p), ops32.shape[0], nthreads)
    if rc != 0:
        raise ValueError("oracle_apply_plan rejected its arguments")


def apply_plan_arrays(direction: str, planes: np.ndarray, host: np.ndarray, ops,
                      nthreads: int = 1) -> None:
    """Same contract as bytes_oracle.apply_plan, on numpy arrays."""
    P, G, chunk = planes.shape
    assert planes.flags.c_contiguous and host.flags.c_contiguous
    base = planes.ctypes.data
    ptrs = [base + p * G * chunk for p in range(P)]
    apply_plan(direction, ptrs, P, chunk, chunk, host.ctypes.data, np.asarray(ops), nthreads)
