"""libkvswap.so (the C ABI of include/kvswap.h) loads on a CPU-only host and
exports every declared symbol; argument validation that never reaches CUDA
returns the documented codes.  No compute calls here (no GPU)."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_2411_18424_b200 import _lib

HEADERS = sorted((Path(__file__).resolve().parents[1] / "include").glob("*.h"))


def declared_symbols():
    found = set()
    for hdr in HEADERS:
        found |= set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(kvs_\w+)\s*\(",
                                hdr.read_text(), re.M))
    return sorted(found)


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(_lib.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for sym in declared_symbols():
        assert hasattr(lib, sym), sym
    assert lib.kvs_abi_version() == 1


def test_error_strings():
    assert _lib.error_string(0) == "ok"
    assert "invalid" in _lib.error_string(_lib.KVS_ERR_INVALID)
    assert "outside" in _lib.error_string(_lib.KVS_ERR_RANGE)
    assert "aligned" in _lib.error_string(_lib.KVS_ERR_ALIGN)


def test_argument_validation_without_gpu():
    lib = _lib.load()
    out = ctypes.c_void_p()
    geo = _lib.KvsGeometry(0, 0, 64, 64)
    ptrs = (ctypes.c_uint64 * 1)(0x1000)
    # bad geometry: zero planes
    assert lib.kvs_create(0, ctypes.byref(geo), ptrs, ctypes.c_void_p(0x2000), 4, 4,
                          ctypes.byref(out)) == _lib.KVS_ERR_INVALID
    # misaligned chunk
    geo = _lib.KvsGeometry(1, 0, 72, 72)
    assert lib.kvs_create(0, ctypes.byref(geo), ptrs, ctypes.c_void_p(0x2000), 4, 4,
                          ctypes.byref(out)) == _lib.KVS_ERR_ALIGN
    # misaligned plane pointer
    geo = _lib.KvsGeometry(1, 0, 64, 64)
    bad = (ctypes.c_uint64 * 1)(0x1008)
    assert lib.kvs_create(0, ctypes.byref(geo), bad, ctypes.c_void_p(0x2000), 4, 4,
                          ctypes.byref(out)) == _lib.KVS_ERR_ALIGN
    # null handle everywhere
    assert lib.kvs_swap(None, 0, None, 0, 0, None, 0) == _lib.KVS_ERR_INVALID
    assert lib.kvs_set_launch(None, 0, 0, 0) == _lib.KVS_ERR_INVALID
    assert lib.kvs_memcpy_baseline(None, 0, 0, None, 0, 0) == _lib.KVS_ERR_INVALID
    assert lib.kvs_launch_count(None) == -1
    assert lib.kvs_destroy(None) == 0
    assert lib.kvs_wait_flag(0, None, 0) == _lib.KVS_ERR_INVALID
    assert lib.kvs_host_free(ctypes.c_void_p(0x1234)) == _lib.KVS_ERR_INVALID
    h, d = ctypes.c_void_p(), ctypes.c_void_p()
    assert lib.kvs_host_alloc(0, -1, 0, ctypes.byref(h), ctypes.byref(d)) == _lib.KVS_ERR_INVALID
    assert lib.kvs_stream_read(0, 0, None, 0, 0, 0, None) == _lib.KVS_ERR_INVALID
    # entry points added for layered admission, pacing priority, SM partition, workload
    sig = _lib.KvsSignals(None, None, None, 1, 0)
    assert lib.kvs_swap_signaled(None, 0, None, 0, 0, ctypes.byref(sig)) == _lib.KVS_ERR_INVALID
    assert lib.kvs_swap_signaled(None, 0, None, 0, 0, None) == _lib.KVS_ERR_INVALID
    assert lib.kvs_swap_ops(None, 0, None, 0, 0, None, None, 0) == _lib.KVS_ERR_INVALID
    assert lib.kvs_swap_layered(None, 0, None, 0, 0, None, 0) == _lib.KVS_ERR_INVALID
    assert lib.kvs_set_layer_group(None, 0) == _lib.KVS_ERR_INVALID
    assert lib.kvs_set_budget_priority(None, 1) == _lib.KVS_ERR_INVALID
    assert lib.kvs_set_pace(None, 0, 1.0) == _lib.KVS_ERR_INVALID
    assert lib.kvs_set_budget(None, 1.0) == _lib.KVS_ERR_INVALID
    assert lib.kvs_set_budget_share(None, 1, 10.0) == _lib.KVS_ERR_INVALID
    assert lib.kvs_set_pace_burst(None, 1, 1 << 20) == _lib.KVS_ERR_INVALID
    assert lib.kvs_set_staging(None, 64 << 20, 4) == _lib.KVS_ERR_INVALID
    assert lib.kvs_set_path(None, 0, 0, 0, 0) == _lib.KVS_ERR_INVALID
    s, r = (ctypes.c_uint64 * 2)(), ctypes.c_uint64()
    sms = (ctypes.c_int * 2)()
    assert lib.kvs_sm_partition(-1, 8, 2, 0, 0, s, ctypes.byref(r), sms) == _lib.KVS_ERR_INVALID
    assert lib.kvs_sm_partition(0, 8, 0, 0, 0, s, ctypes.byref(r), sms) == _lib.KVS_ERR_INVALID
    assert lib.kvs_kv_tokens(None, 0, None, 0, 16, 0, -1, 0, None) == _lib.KVS_ERR_INVALID
    step = _lib.KvsDecodeStep()
    how = ctypes.c_int()
    assert lib.kvs_graph_decode_step(None, None, ctypes.byref(step), ctypes.byref(how)) == \
        _lib.KVS_ERR_INVALID


def test_check_maps_codes_to_reference_exceptions():
    with pytest.raises(ValueError):
        _lib.check(_lib.KVS_ERR_INVALID)
    with pytest.raises(IndexError):
        _lib.check(_lib.KVS_ERR_RANGE)
    with pytest.raises(MemoryError):
        _lib.check(_lib.KVS_ERR_NOMEM)
    with pytest.raises(_lib.KvSwapCudaError):
        _lib.check(2)  # cudaErrorMemoryAllocation
    _lib.check(0)


def test_missing_library_fails_loudly(tmp_path):
    with pytest.raises(_lib.NativeLibraryError):
        _lib.load(tmp_path / "libkvswap.so")
