"""ctypes binding of the control plane's C ABI (include/kvctrl.h, libkvctrl.so).

This is what a non-CPython host binds; inside this
package the engine uses the CPython extension `_kvctrl` over the same C++
(native_ctrl.py).  This module exposes exactly the extension's function
surface (`pool_allocate(handle, ...)`, `store_plan_swap_out(...)`, ...) on
top of the C ABI, so `NativeBlockGroupPool(cfg, backend=kvctrl_cabi)` runs the
same classes over the C ABI and tests/test_native_ctrl.py checks both
bindings with the same differential fuzz and goldens.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libkvctrl.so"
NONE = -(1 << 63)  # KVC_NONE

# every symbol include/kvctrl.h declares
EXPORTS = [
    "kvc_abi_version", "kvc_last_error", "kvc_rng_draws",
    "kvc_pool_create", "kvc_pool_destroy", "kvc_pool_set_rank_fn", "kvc_pool_allocate",
    "kvc_pool_reclaim_from_victim", "kvc_pool_allocate_at", "kvc_pool_free_group",
    "kvc_pool_shrink_group", "kvc_pool_free_request", "kvc_pool_set_request_fill",
    "kvc_pool_record_transfer", "kvc_pool_counters", "kvc_pool_owned_blocks",
    "kvc_pool_reclaimable_blocks", "kvc_pool_group", "kvc_pool_owned_groups",
    "kvc_pool_free_groups", "kvc_pool_extents", "kvc_pool_set_group_filled",
    "kvc_pool_granularity", "kvc_pool_dump", "kvc_pool_validate",
    "kvc_store_create", "kvc_store_destroy", "kvc_store_pool", "kvc_store_set_flag",
    "kvc_store_counters", "kvc_store_set_rank", "kvc_store_set_ranks", "kvc_store_get_rank",
    "kvc_store_del_rank", "kvc_store_ranks", "kvc_store_clear_ranks",
    "kvc_store_plan_swap_out", "kvc_store_plan_swap_in", "kvc_store_plan_swap_in_prefix",
    "kvc_store_evict_for", "kvc_store_preallocate_increment", "kvc_store_release",
    "kvc_store_ensure_free", "kvc_store_track_peak", "kvc_store_copy_ids", "kvc_store_copy",
    "kvc_store_put_copy", "kvc_store_drop_copy",
]

RANK_FN = C.CFUNCTYPE(C.c_int64, C.c_void_p, C.c_int64)
_P64 = C.POINTER(C.c_int64)
_lib = None
_errors: dict[int, type] = {}


class NativeLibraryError(RuntimeError):
    """libkvctrl.so is missing or does not match include/kvctrl.h."""


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise NativeLibraryError(f"{LIB_PATH} not built (run __graft_entry__.build())")
    lib = C.CDLL(str(LIB_PATH))
    missing = [s for s in EXPORTS if not hasattr(lib, s)]
    if missing:
        raise NativeLibraryError(f"libkvctrl.so lacks {missing}")
    if lib.kvc_abi_version() != 1:
        raise NativeLibraryError("libkvctrl.so ABI version mismatch")
    vp, i64, i32, ci = C.c_void_p, C.c_int64, C.c_int32, C.c_int
    res = [C.POINTER(_P64), _P64]
    sig = {
        "kvc_last_error": ([], C.c_char_p),
        "kvc_rng_draws": ([_P64, i32, i64, i64, _P64], ci),
        "kvc_pool_create": ([i64, i64, i64, ci, C.POINTER(vp)], ci),
        "kvc_pool_destroy": ([vp], ci),
        "kvc_pool_set_rank_fn": ([vp, RANK_FN, vp], ci),
        "kvc_pool_allocate": ([vp, i64, i64, i64, ci] + res, ci),
        "kvc_pool_reclaim_from_victim": ([vp, i64, i64] + res, ci),
        "kvc_pool_allocate_at": ([vp, i64, i64, i64] + res, ci),
        "kvc_pool_free_group": ([vp, i64], ci),
        "kvc_pool_shrink_group": ([vp, i64, i64], ci),
        "kvc_pool_free_request": ([vp, i64, _P64], ci),
        "kvc_pool_set_request_fill": ([vp, i64, i64], ci),
        "kvc_pool_record_transfer": ([vp, i64], ci),
        "kvc_pool_counters": ([vp, _P64], ci),
        "kvc_pool_owned_blocks": ([vp, i64, _P64], ci),
        "kvc_pool_reclaimable_blocks": ([vp, i64, _P64], ci),
        "kvc_pool_group": ([vp, i64, _P64], ci),
        "kvc_pool_owned_groups": ([vp, i64] + res, ci),
        "kvc_pool_free_groups": ([vp] + res, ci),
        "kvc_pool_extents": ([vp, i64] + res, ci),
        "kvc_pool_set_group_filled": ([vp, i64, i64], ci),
        "kvc_pool_granularity": ([vp] + res, ci),
        "kvc_pool_dump": ([vp, C.c_char_p, i64, _P64], ci),
        "kvc_pool_validate": ([vp], ci),
        "kvc_store_create": ([i64, ci, i64, i64, ci, i64, C.POINTER(vp)], ci),
        "kvc_store_destroy": ([vp], ci),
        "kvc_store_pool": ([vp, C.POINTER(vp)], ci),
        "kvc_store_set_flag": ([vp, ci, i64], ci),
        "kvc_store_counters": ([vp, _P64], ci),
        "kvc_store_set_rank": ([vp, i64, i64], ci),
        "kvc_store_set_ranks": ([vp, _P64, i64], ci),
        "kvc_store_get_rank": ([vp, i64, _P64], ci),
        "kvc_store_del_rank": ([vp, i64], ci),
        "kvc_store_ranks": ([vp] + res, ci),
        "kvc_store_clear_ranks": ([vp], ci),
        "kvc_store_plan_swap_out": ([vp, i64, i64, _P64, i64, i64] + res, ci),
        "kvc_store_plan_swap_in": ([vp, i64, _P64, i64] + res, ci),
        "kvc_store_plan_swap_in_prefix": ([vp, i64, _P64, i64] + res, ci),
        "kvc_store_evict_for": ([vp, i64, i64] + res, ci),
        "kvc_store_preallocate_increment": ([vp, i64, i64, C.POINTER(ci)], ci),
        "kvc_store_release": ([vp, i64], ci),
        "kvc_store_ensure_free": ([vp, i64, i64], ci),
        "kvc_store_track_peak": ([vp], ci),
        "kvc_store_copy_ids": ([vp] + res, ci),
        "kvc_store_copy": ([vp, i64] + res, ci),
        "kvc_store_put_copy": ([vp, i64, i64, i64, _P64, i64], ci),
        "kvc_store_drop_copy": ([vp, i64], ci),
    }
    for name, (args, ret) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ret
    _lib = lib
    return lib


def set_exceptions(pool_error, oom, no_victim, cpu_oom, contaminated, insufficient) -> None:
    _errors.update({-10: pool_error, -11: oom, -12: no_victim, -13: ValueError, -14: KeyError,
                    -15: AssertionError, -16: cpu_oom, -17: contaminated, -18: insufficient,
                    -19: StopIteration})


def _check(rc: int) -> None:
    if rc:
        raise _errors.get(rc, RuntimeError)(_lib.kvc_last_error().decode())


def _opt(v) -> int:
    return NONE if v is None else int(v)


def _py(v: int):
    return None if v == NONE else v


def _arr(values):
    values = list(values)
    return (C.c_int64 * max(1, len(values)))(*values)


class _Handle:
    """Owns (or borrows) a C handle; destroys it with the matching call."""

    def __init__(self, ptr, destroy=None, keep=None) -> None:
        self.ptr = ptr
        self._destroy = destroy
        self._keep = keep
        self.rank_cb = None
        self.res_ptr = _P64()
        self.res_n = C.c_int64()

    def res(self):
        return C.byref(self.res_ptr), C.byref(self.res_n)

    def words(self) -> list[int]:
        n = self.res_n.value
        return self.res_ptr[:n] if n else []

    def __del__(self) -> None:
        if self._destroy is not None and _lib is not None and self.ptr:
            getattr(_lib, self._destroy)(self.ptr)
            self.ptr = None


def _call(h: _Handle, name: str, *args):
    _check(getattr(_lib, name)(h.ptr, *args, *h.res()))
    return h.words()


def _g7(w, i=0):
    return (w[i], w[i + 1], w[i + 2], bool(w[i + 3]), _py(w[i + 4]), bool(w[i + 5]), w[i + 6])


def _plan(w):
    n, nr = w[2], w[3]
    ops = [tuple(w[j:j + 3]) for j in range(4, 4 + 3 * n, 3)]
    ref = [tuple(w[j:j + 3]) for j in range(4 + 3 * n, 4 + 3 * (n + nr), 3)]
    return w[0], w[1], ops, ref


def _ext(extents):
    flat = [v for e in extents for v in e]
    return _arr(flat), len(flat) // 2


# ---------------------------------------------------------------- functions
def rng_draws(entropy, bound, n):
    out = (C.c_int64 * max(1, n))()
    _check(_lib.kvc_rng_draws(_arr(entropy), len(entropy), bound, n, out))
    return list(out)[:n]


def pool_create(total, initial, seed, policy):
    h = C.c_void_p()
    _check(_lib.kvc_pool_create(total, initial, seed, policy, C.byref(h)))
    return _Handle(h, "kvc_pool_destroy")


def pool_set_rank_fn(h, fn):
    h.rank_cb = RANK_FN(lambda _ctx, req: int(fn(req))) if fn is not None else RANK_FN()
    _check(_lib.kvc_pool_set_rank_fn(h.ptr, h.rank_cb, None))


def pool_allocate(h, req, want, expected, reclaim):
    w = _call(h, "kvc_pool_allocate", req, want, _opt(expected), 1 if reclaim else 0)
    ng, nc = w[0], w[1]
    groups = [tuple(w[j:j + 3]) for j in range(2, 2 + 3 * ng, 3)]
    at = 2 + 3 * ng
    return groups, [(w[j], w[j + 1]) for j in range(at, at + 2 * nc, 2)]


def pool_reclaim_from_victim(h, need, for_request):
    return tuple(_call(h, "kvc_pool_reclaim_from_victim", need, for_request))


def pool_allocate_at(h, req, start, length):
    w = _call(h, "kvc_pool_allocate_at", req, start, length)
    return tuple(w) if w else None


def pool_free_group(h, gid):
    _check(_lib.kvc_pool_free_group(h.ptr, gid))


def pool_shrink_group(h, gid, n):
    _check(_lib.kvc_pool_shrink_group(h.ptr, gid, n))


def pool_free_request(h, req):
    out = C.c_int64()
    _check(_lib.kvc_pool_free_request(h.ptr, req, C.byref(out)))
    return out.value


def pool_set_request_fill(h, req, n):
    _check(_lib.kvc_pool_set_request_fill(h.ptr, req, n))


def pool_record_transfer(h, blocks):
    _check(_lib.kvc_pool_record_transfer(h.ptr, blocks))


def pool_counters(h):
    out = (C.c_int64 * 6)()
    _check(_lib.kvc_pool_counters(h.ptr, out))
    return tuple(out)


def pool_free_blocks(h):
    return pool_counters(h)[1]


def pool_owned_blocks(h, req):
    out = C.c_int64()
    _check(_lib.kvc_pool_owned_blocks(h.ptr, req, C.byref(out)))
    return out.value


def pool_reclaimable(h, exclude):
    out = C.c_int64()
    _check(_lib.kvc_pool_reclaimable_blocks(h.ptr, _opt(exclude), C.byref(out)))
    return out.value


def pool_group(h, gid):
    out = (C.c_int64 * 7)()
    _check(_lib.kvc_pool_group(h.ptr, gid, out))
    return _g7(list(out))


def pool_owned_groups(h, req):
    w = _call(h, "kvc_pool_owned_groups", req)
    return [_g7(w, i) for i in range(0, len(w), 7)]


def pool_free_groups(h):
    w = _call(h, "kvc_pool_free_groups")
    return [_g7(w, i) for i in range(0, len(w), 7)]


def pool_extents(h, req):
    w = _call(h, "kvc_pool_extents", req)
    return [(w[i], w[i + 1]) for i in range(0, len(w), 2)]


def pool_granularity(h):
    w = _call(h, "kvc_pool_granularity")
    return {w[i]: w[i + 1] for i in range(0, len(w), 2)}


def pool_dump(h):
    need = C.c_int64()
    _check(_lib.kvc_pool_dump(h.ptr, None, 0, C.byref(need)))
    buf = C.create_string_buffer(need.value)
    _check(_lib.kvc_pool_dump(h.ptr, buf, need.value, C.byref(need)))
    return buf.value.decode()


def pool_validate(h):
    _check(_lib.kvc_pool_validate(h.ptr))


def store_create(total, reuse, pmin, pmax, rel, bt):
    h = C.c_void_p()
    _check(_lib.kvc_store_create(total, reuse, pmin, pmax, rel, bt, C.byref(h)))
    return _Handle(h, "kvc_store_destroy")


def store_pool(h):
    p = C.c_void_p()
    _check(_lib.kvc_store_pool(h.ptr, C.byref(p)))
    return _Handle(p, None, keep=h)


def store_set_flag(h, which, v):
    _check(_lib.kvc_store_set_flag(h.ptr, which, v))


def store_counters(h):
    out = (C.c_int64 * 5)()
    _check(_lib.kvc_store_counters(h.ptr, out))
    return tuple(out)


def store_set_rank(h, req, rank):
    _check(_lib.kvc_store_set_rank(h.ptr, req, rank))


def store_set_ranks(h, ranks):
    flat = [v for kv in ranks.items() for v in kv]
    _check(_lib.kvc_store_set_ranks(h.ptr, _arr(flat), len(ranks)))


def store_get_rank(h, req):
    out = C.c_int64()
    _check(_lib.kvc_store_get_rank(h.ptr, req, C.byref(out)))
    return _py(out.value)


def store_del_rank(h, req):
    _check(_lib.kvc_store_del_rank(h.ptr, req))


def store_ranks(h):
    w = _call(h, "kvc_store_ranks")
    return [(w[i], w[i + 1]) for i in range(0, len(w), 2)]


def store_clear_ranks(h):
    _check(_lib.kvc_store_clear_ranks(h.ptr))


def store_plan_swap_out(h, req, fp, extents, tokens):
    ext, n = _ext(extents)
    return _plan(_call(h, "kvc_store_plan_swap_out", req, fp, ext, n, _opt(tokens)))


def store_plan_swap_in(h, req, extents):
    ext, n = _ext(extents)
    return _plan(_call(h, "kvc_store_plan_swap_in", req, ext, n))


def store_plan_swap_in_prefix(h, req, extents):
    ext, n = _ext(extents)
    w = _call(h, "kvc_store_plan_swap_in_prefix", req, ext, n)
    return _plan(w), w[-1]


def store_evict_for(h, rank, need):
    w = _call(h, "kvc_store_evict_for", rank, need)
    return [(w[i], w[i + 1]) for i in range(0, len(w), 2)]


def store_preallocate_increment(h, req, inc):
    ok = C.c_int()
    _check(_lib.kvc_store_preallocate_increment(h.ptr, req, inc, C.byref(ok)))
    return bool(ok.value)


def store_release(h, req):
    _check(_lib.kvc_store_release(h.ptr, req))


def store_ensure_free(h, req, need):
    _check(_lib.kvc_store_ensure_free(h.ptr, req, need))


def store_track_peak(h):
    _check(_lib.kvc_store_track_peak(h.ptr))


def store_copy_ids(h):
    return list(_call(h, "kvc_store_copy_ids"))


def store_has_copy(h, req):
    return req in store_copy_ids(h)


def store_copy(h, req):
    w = _call(h, "kvc_store_copy", req)
    segs = [(w[j], w[j + 1], _py(w[j + 2]), bool(w[j + 3])) for j in range(3, 3 + 4 * w[2], 4)]
    return _py(w[0]), _py(w[1]), segs


def store_put_copy(h, req, prealloc, saved, segs):
    flat = [v for lo, hi, gid, ok in segs for v in (lo, hi, _opt(gid), 1 if ok else 0)]
    _check(_lib.kvc_store_put_copy(h.ptr, req, _opt(prealloc), _opt(saved), _arr(flat),
                                   len(segs)))


def store_drop_copy(h, req):
    _check(_lib.kvc_store_drop_copy(h.ptr, req))
