"""Native control plane: the reference's block-group
allocator and CPU store in C++ (csrc/ctrlplane.cpp), behind the reference's
Python API.

`NativeBlockGroupPool` is a drop-in for kvswitch.alloc.BlockGroupPool
(pkg/src/kvswitch/alloc.py:95-532) and `NativeCpuStore` for
kvswitch.cpu_store.CpuStore (pkg/src/kvswitch/cpu_store.py:123-403): same
constructor arguments, methods, return types and exceptions, and every
decision — group ids, block tables, the seeded random victim draws (numpy
PCG64 restated in C++), plans, evictions — is bit-exact with the reference
(tests/test_native_ctrl.py: differential fuzz against the Python control
plane, the reference's own unit tests, the engine replay goldens).
`Engine(..., control_plane="native")` runs on it.

Bindings.  The engine calls the CPython extension `_kvctrl`
(csrc/kvctrl_py.cpp, METH_FASTCALL: ~0.1 µs per call); `backend=kvctrl_cabi`
runs the same classes over the C ABI (include/kvctrl.h, libkvctrl.so,
ctypes) — what a non-Python host would bind.  Both are built from the same
C++ and checked by the same tests.

Objects handed out are snapshots (`BlockGroup`) or write-through views (a
CPU copy and its segments, `store.copies`, `store.ranks`), so the reference's
tests that edit a copy's segments in place work unchanged.  There is no
Python fallback: a missing extension raises NativeLibraryError.
"""

from __future__ import annotations

import importlib
from collections.abc import MutableMapping
from typing import Callable, Optional

from .alloc import (AllocResult, BlockGroup, NoVictimError, OutOfMemoryError, PoolConfig,
                    PoolError)
from .cpu_store import (ContaminatedCopyError, CpuOutOfMemoryError, InsufficientVictimsError,
                        Segment, SwapPlan, TransferOp)


class NativeLibraryError(RuntimeError):
    """The native control plane (_kvctrl / libkvctrl.so) is not built."""


_EXC = (PoolError, OutOfMemoryError, NoVictimError, CpuOutOfMemoryError, ContaminatedCopyError,
        InsufficientVictimsError)
_ext = None


def load():
    """The CPython extension (built by _build.build_kvctrl)."""
    global _ext
    if _ext is None:
        try:
            mod = importlib.import_module("paper_2411_18424_b200._kvctrl")
        except ImportError as exc:
            raise NativeLibraryError(
                "paper_2411_18424_b200/_kvctrl*.so not built (run __graft_entry__.build())"
            ) from exc
        mod.set_exceptions(*_EXC)
        _ext = mod
    return _ext


def cabi_backend():
    """The ctypes binding of include/kvctrl.h, with this module's exceptions."""
    from . import kvctrl_cabi
    kvctrl_cabi.load()
    kvctrl_cabi.set_exceptions(*_EXC)
    return kvctrl_cabi


_new = object.__new__


def _group(t) -> BlockGroup:
    g = _new(BlockGroup)  # field-for-field BlockGroup without the dataclass __init__
    g.__dict__.update(id=t[0], start=t[1], length=t[2], free=t[3], owner=t[4], active=t[5],
                      filled=t[6])
    return g


def _used(gid: int, start: int, length: int, owner: int, active: bool) -> BlockGroup:
    g = _new(BlockGroup)
    g.__dict__.update(id=gid, start=start, length=length, free=False, owner=owner,
                      active=active, filled=0)
    return g


def _op(t) -> TransferOp:
    o = _new(TransferOp)  # frozen dataclass: fill its fields without __setattr__
    o.__dict__.update(blocks=t[0], gpu_start=t[1], cpu_start=t[2])
    return o


# ---------------------------------------------------------------------------
class NativeBlockGroupPool:
    """kvswitch.alloc.BlockGroupPool on the native control plane."""

    def __init__(self, config: PoolConfig, backend=None, _handle=None) -> None:
        self._b = backend or load()
        self.config = config
        self.total_blocks = config.total_blocks
        if _handle is None:
            _handle = self._b.pool_create(
                config.total_blocks, config.initial_group_blocks, config.rng_seed,
                1 if config.victim_policy == "lowest_priority" else 0)
        self._h = _handle
        self._rank_of: Optional[Callable[[int], int]] = None

    # -- priority hook (alloc.py:310-315) --------------------------------------
    @property
    def rank_of(self) -> Optional[Callable[[int], int]]:
        return self._rank_of

    @rank_of.setter
    def rank_of(self, fn: Optional[Callable[[int], int]]) -> None:
        self._rank_of = fn
        self._b.pool_set_rank_fn(self._h, fn)

    # -- queries -----------------------------------------------------------------
    @property
    def free_blocks(self) -> int:
        return self._b.pool_free_blocks(self._h)

    @property
    def used_blocks(self) -> int:
        return self.total_blocks - self._b.pool_free_blocks(self._h)

    def group(self, gid: int) -> BlockGroup:
        return _group(self._b.pool_group(self._h, gid))

    def owned_groups(self, req: int) -> list[BlockGroup]:
        return [_group(t) for t in self._b.pool_owned_groups(self._h, req)]

    def owned_blocks(self, req: int) -> int:
        return self._b.pool_owned_blocks(self._h, req)

    def free_groups(self) -> list[BlockGroup]:
        return [_group(t) for t in self._b.pool_free_groups(self._h)]

    def reclaimable_blocks(self, exclude: Optional[int] = None) -> int:
        return self._b.pool_reclaimable(self._h, exclude)

    def extents(self, req: int) -> list[tuple[int, int]]:
        """The block table (engine.py:317-325) in one call."""
        return self._b.pool_extents(self._h, req)

    # -- allocation ----------------------------------------------------------------
    def allocate(self, req: int, want_blocks: int, expected_total: Optional[int] = None,
                 reclaim: bool = True) -> AllocResult:
        grants, carved = self._b.pool_allocate(self._h, req, want_blocks, expected_total,
                                               reclaim)
        groups = [_used(g, s, n, req, False) for g, s, n in grants]
        groups[-1].active = True
        return AllocResult(groups=groups, reclaimed_from=carved)

    def reclaim_from_victim(self, need_blocks: int, *,
                            for_request: int) -> tuple[int, BlockGroup]:
        owner, gid, start, length = self._b.pool_reclaim_from_victim(self._h, need_blocks,
                                                                     for_request)
        return owner, BlockGroup(id=gid, start=start, length=length, free=False,
                                 owner=for_request, active=True)

    def allocate_at(self, req: int, start: int, length: int) -> Optional[BlockGroup]:
        t = self._b.pool_allocate_at(self._h, req, start, length)
        if t is None:
            return None
        return BlockGroup(id=t[0], start=t[1], length=t[2], free=False, owner=req, active=True)

    # -- release ---------------------------------------------------------------------
    def free_group(self, gid: int) -> None:
        self._b.pool_free_group(self._h, gid)

    def shrink_group(self, gid: int, new_length: int) -> None:
        self._b.pool_shrink_group(self._h, gid, new_length)

    def free_request(self, req: int) -> int:
        return self._b.pool_free_request(self._h, req)

    def set_request_fill(self, req: int, filled_blocks: int) -> None:
        self._b.pool_set_request_fill(self._h, req, filled_blocks)

    # -- transfer granularity ----------------------------------------------------------
    def record_transfer(self, blocks: int) -> None:
        self._b.pool_record_transfer(self._h, blocks)

    def granularity_stats(self) -> Optional[tuple[float, dict[int, int]]]:
        c = self._b.pool_counters(self._h)
        if not c[4]:
            return None
        return c[5] / c[4], self._b.pool_granularity(self._h)

    # -- debugging -----------------------------------------------------------------------
    def dump(self) -> str:
        return self._b.pool_dump(self._h)

    def validate(self) -> None:
        self._b.pool_validate(self._h)


# ---------------------------------------------------------------------------
class _NativeSegment:
    """Write-through view of segment `i` of a native CPU copy."""

    __slots__ = ("_copy", "_i")

    def __init__(self, copy: "NativeCpuCopy", i: int) -> None:
        self._copy = copy
        self._i = i

    def _get(self, k: int):
        return self._copy._read()[2][self._i][k]

    def _set(self, k: int, v) -> None:
        pre, saved, segs = self._copy._read()
        row = list(segs[self._i])
        row[k] = v
        segs[self._i] = tuple(row)
        self._copy._write(pre, saved, segs)

    block_lo = property(lambda s: s._get(0), lambda s, v: s._set(0, int(v)))
    block_hi = property(lambda s: s._get(1), lambda s, v: s._set(1, int(v)))
    group_id = property(lambda s: s._get(2), lambda s, v: s._set(2, v))
    valid = property(lambda s: s._get(3), lambda s, v: s._set(3, bool(v)))

    @property
    def length(self) -> int:
        lo, hi = self._copy._read()[2][self._i][:2]
        return hi - lo

    def __repr__(self) -> str:
        return "Segment(block_lo=%r, block_hi=%r, group_id=%r, valid=%r)" % \
            self._copy._read()[2][self._i]

    def __eq__(self, other) -> bool:
        return all(getattr(self, k) == getattr(other, k, None)
                   for k in ("block_lo", "block_hi", "group_id", "valid"))


class NativeCpuCopy:
    """Write-through view of one request's CPU copy (cpu_store.py:31-70)."""

    def __init__(self, store: "NativeCpuStore", owner: int) -> None:
        self._store = store
        self.owner = owner

    def _read(self):
        return self._store._b.store_copy(self._store._h, self.owner)

    def _write(self, prealloc, saved, segs) -> None:
        self._store._b.store_put_copy(self._store._h, self.owner, prealloc, saved, segs)

    @property
    def segments(self) -> list[_NativeSegment]:
        return [_NativeSegment(self, i) for i in range(len(self._read()[2]))]

    @segments.setter
    def segments(self, segs) -> None:
        pre, saved, _ = self._read()
        self._write(pre, saved, [(s.block_lo, s.block_hi, s.group_id, s.valid) for s in segs])

    @property
    def prealloc(self) -> Optional[int]:
        return self._read()[0]

    @prealloc.setter
    def prealloc(self, gid: Optional[int]) -> None:
        _, saved, segs = self._read()
        self._write(gid, saved, segs)

    @property
    def saved_tokens(self) -> Optional[int]:
        return self._read()[1]

    @saved_tokens.setter
    def saved_tokens(self, tokens: Optional[int]) -> None:
        pre, _, segs = self._read()
        self._write(pre, tokens, segs)

    @property
    def covered_blocks(self) -> int:
        segs = self._read()[2]
        return segs[-1][1] if segs else 0

    @property
    def valid_blocks(self) -> int:
        return sum(hi - lo for lo, hi, _, ok in self._read()[2] if ok)

    @property
    def fully_valid(self) -> bool:
        return all(ok for _, _, _, ok in self._read()[2])

    def valid_prefix_blocks(self) -> int:
        reach = 0
        for lo, hi, _, ok in self._read()[2]:
            if not (ok and lo == reach):
                return reach
            reach = hi
        return reach


class _Copies(MutableMapping):
    """store.copies: request -> NativeCpuCopy view."""

    def __init__(self, store: "NativeCpuStore") -> None:
        self._s = store

    def __getitem__(self, req: int) -> NativeCpuCopy:
        if not self._s._b.store_has_copy(self._s._h, req):
            raise KeyError(req)
        return NativeCpuCopy(self._s, req)

    def __setitem__(self, req: int, copy) -> None:
        self._s._b.store_put_copy(
            self._s._h, req, copy.prealloc, copy.saved_tokens,
            [(s.block_lo, s.block_hi, s.group_id, s.valid) for s in copy.segments])

    def __delitem__(self, req: int) -> None:
        self._s._b.store_drop_copy(self._s._h, req)

    def __iter__(self):
        return iter(self._s._b.store_copy_ids(self._s._h))

    def __len__(self) -> int:
        return self._s._b.store_counters(self._s._h)[2]

    def __contains__(self, req) -> bool:
        return self._s._b.store_has_copy(self._s._h, req)


class _Ranks(MutableMapping):
    """store.ranks: request -> priority rank, held natively."""

    def __init__(self, store: "NativeCpuStore") -> None:
        self._s = store

    def __getitem__(self, req: int) -> int:
        r = self._s._b.store_get_rank(self._s._h, req)
        if r is None:
            raise KeyError(req)
        return r

    def get(self, req, default=None):
        r = self._s._b.store_get_rank(self._s._h, req)
        return default if r is None else r

    def __setitem__(self, req: int, rank: int) -> None:
        self._s._b.store_set_rank(self._s._h, req, rank)

    def __delitem__(self, req: int) -> None:
        self._s._b.store_del_rank(self._s._h, req)

    def __iter__(self):
        return iter([r for r, _ in self._s._b.store_ranks(self._s._h)])

    def __len__(self) -> int:
        return self._s._b.store_counters(self._s._h)[3]

    def __contains__(self, req) -> bool:
        return self._s._b.store_get_rank(self._s._h, req) is not None

    def update(self, other=(), **kw) -> None:
        d = dict(other)
        d.update(kw)
        self._s._b.store_set_ranks(self._s._h, d)

    def clear(self) -> None:
        self._s._b.store_clear_ranks(self._s._h)


class NativeCpuStore:
    """kvswitch.cpu_store.CpuStore on the native control plane, plus the
    dirty-tail refresh op of the package's CpuStore."""

    def __init__(self, total_blocks: int, reuse_enabled: bool = True,
                 prealloc_min_blocks: int = 8, prealloc_max_blocks: int = 256,
                 release_on_swap_in: bool = False, block_size_tokens: int = 16,
                 backend=None) -> None:
        self._b = backend or load()
        self._h = self._b.store_create(total_blocks, 1 if reuse_enabled else 0,
                                       prealloc_min_blocks, prealloc_max_blocks,
                                       1 if release_on_swap_in else 0, block_size_tokens)
        self.pool = NativeBlockGroupPool(
            PoolConfig(total_blocks=total_blocks, initial_group_blocks=1), backend=self._b,
            _handle=self._b.store_pool(self._h))
        self._reuse = reuse_enabled
        self._release = release_on_swap_in
        self.prealloc_min_blocks = prealloc_min_blocks
        self.prealloc_max_blocks = prealloc_max_blocks
        self.block_size_tokens = block_size_tokens
        self.copies = _Copies(self)
        self.ranks = _Ranks(self)

    # -- flags and counters ------------------------------------------------------
    @property
    def reuse_enabled(self) -> bool:
        return self._reuse

    @reuse_enabled.setter
    def reuse_enabled(self, on: bool) -> None:
        self._b.store_set_flag(self._h, 0, 1 if on else 0)
        self._reuse = bool(on)

    @property
    def release_on_swap_in(self) -> bool:
        return self._release

    @release_on_swap_in.setter
    def release_on_swap_in(self, on: bool) -> None:
        self._b.store_set_flag(self._h, 2, 1 if on else 0)
        self._release = bool(on)

    @property
    def refresh_dirty_tail(self) -> bool:
        return bool(self._b.store_counters(self._h)[4])

    @refresh_dirty_tail.setter
    def refresh_dirty_tail(self, on: bool) -> None:
        self._b.store_set_flag(self._h, 1, 1 if on else 0)

    @property
    def peak_used_blocks(self) -> int:
        return self._b.store_counters(self._h)[0]

    @property
    def refreshed_blocks(self) -> int:
        return self._b.store_counters(self._h)[1]

    # -- priorities -------------------------------------------------------------------
    def set_rank(self, req: int, rank: int) -> None:
        self._b.store_set_rank(self._h, req, rank)

    def update_ranks(self, ranks: dict[int, int]) -> None:
        self._b.store_set_ranks(self._h, ranks)

    def copy_of(self, req: int) -> Optional[NativeCpuCopy]:
        return NativeCpuCopy(self, req) if self._b.store_has_copy(self._h, req) else None

    # -- plans --------------------------------------------------------------------------
    @staticmethod
    def _plan(req: int, direction: str, t) -> SwapPlan:
        moved, reused, ops, refresh = t
        return SwapPlan(req, direction, [_op(o) for o in ops], moved, reused,
                        [_op(o) for o in refresh] if refresh else [])

    def plan_swap_out(self, req: int, gpu_footprint: int, gpu_extents: list[tuple[int, int]],
                      tokens: Optional[int] = None) -> SwapPlan:
        return self._plan(req, "out", self._b.store_plan_swap_out(self._h, req, gpu_footprint,
                                                                  gpu_extents, tokens))

    def plan_swap_in(self, req: int, gpu_extents: list[tuple[int, int]]) -> SwapPlan:
        return self._plan(req, "in", self._b.store_plan_swap_in(self._h, req, gpu_extents))

    def plan_swap_in_prefix(self, req: int,
                            gpu_extents: list[tuple[int, int]]) -> tuple[SwapPlan, int]:
        t, keep = self._b.store_plan_swap_in_prefix(self._h, req, gpu_extents)
        return self._plan(req, "in", t), keep

    # -- eviction / reservation -------------------------------------------------------
    def evict_for(self, rank: int, need_blocks: int) -> list[tuple[int, int]]:
        return self._b.store_evict_for(self._h, rank, need_blocks)

    def preallocate_increment(self, req: int, expected_increment: int) -> bool:
        return self._b.store_preallocate_increment(self._h, req, expected_increment)

    def release(self, req: int) -> None:
        self._b.store_release(self._h, req)

    def _ensure_free(self, req: int, need: int) -> None:
        self._b.store_ensure_free(self._h, req, need)

    def _track_peak(self) -> None:
        self._b.store_track_peak(self._h)

    def _host_extents(self, copy) -> list[tuple[int, int, int]]:
        """Backed segments as fused logical extents (cpu_store.py:169-180)."""
        out: list[tuple[int, int, int]] = []
        for s in copy.segments:
            if s.group_id is None:
                continue
            phys = self.pool.group(s.group_id).start
            if out:
                lo, hi, base = out[-1]
                if hi == s.block_lo and base + (hi - lo) == phys:
                    out[-1] = (lo, s.block_hi, base)
                    continue
            out.append((s.block_lo, s.block_hi, phys))
        return out

    _logical_extents = _host_extents

    def dump(self) -> str:
        return "\n".join("cpu " + line for line in self.pool.dump().splitlines())


__all__ = ["NativeBlockGroupPool", "NativeCpuStore", "NativeCpuCopy", "NativeLibraryError",
           "Segment", "load", "cabi_backend"]
