"""Native control plane: the C++ block-group pool and
CPU store (csrc/ctrlplane.cpp) behind the reference's Python API
(native_ctrl.py), through both bindings — the CPython extension the engine
uses and the C ABI (include/kvctrl.h) over ctypes.

Parity is pinned three ways, all on CPU:
  * differential fuzz against the package's Python control plane (itself
    pinned to the reference): every return value, exception class, pool dump,
    copy segment list, rank map and counter after every operation;
  * the reference's golden op sequences and all engine replay goldens
    (tests/golden/, recorded from the unmodified reference) with
    control_plane="native";
  * the reference's own unit tests run against the native classes.
"""

import random
import subprocess
import sys
import types
from pathlib import Path

import numpy as np
import pytest

from oracle import gen_golden as gg
from paper_2411_18424_b200 import alloc, cpu_store, engine, native_ctrl
from paper_2411_18424_b200.alloc import AllocResult, BlockGroup, BlockGroupPool, PoolConfig
from paper_2411_18424_b200.cpu_store import CpuStore, SwapPlan

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tests"))
import test_golden as tg  # noqa: E402

BACKENDS = ["ext", "cabi"]


def backend(name):
    return native_ctrl.load() if name == "ext" else native_ctrl.cabi_backend()


def test_bindings_load_and_export_every_symbol():
    from paper_2411_18424_b200 import kvctrl_cabi
    native_ctrl.load()
    lib = kvctrl_cabi.load()
    header = (ROOT / "include" / "kvctrl.h").read_text()
    import re
    declared = set(re.findall(r"^(?:int|const char\*)\s+(kvc_\w+)\(", header, re.M))
    assert declared == set(kvctrl_cabi.EXPORTS)
    for sym in declared:
        assert hasattr(lib, sym), sym


@pytest.mark.parametrize("be", BACKENDS)
def test_victim_rng_is_numpy_pcg64(be):
    """The random victim policy draws Generator(PCG64(SeedSequence([seed,
    0x6A11]))).integers(n) (alloc.py:101, :314), bit for bit."""
    b = backend(be)
    for ent in ([0, 0x6A11], [12345, 0x6A11], [2**40 + 7, 3], [7, 8, 9, 10, 11, 12]):
        for bound in (1, 2, 3, 7, 100, 2**31 + 5, 2**32, 2**40 + 3):
            r = np.random.default_rng(np.random.SeedSequence(ent))
            assert b.rng_draws(ent, bound, 40) == [int(r.integers(bound)) for _ in range(40)]


# ---------------------------------------------------------------- fuzz
def _norm(r):
    if isinstance(r, AllocResult):
        return ([(g.id, g.start, g.length) for g in r.groups], r.reclaimed_from)
    if isinstance(r, BlockGroup):
        return (r.id, r.start, r.length)
    if isinstance(r, SwapPlan):
        return (r.request, r.direction, [(o.blocks, o.gpu_start, o.cpu_start) for o in r.ops],
                r.moved_blocks, r.reused_blocks,
                [(o.blocks, o.gpu_start, o.cpu_start) for o in r.refresh_ops])
    if isinstance(r, tuple):
        return tuple(_norm(x) for x in r)
    return r


def _call(obj, name, *a, **k):
    try:
        return ("ok", _norm(getattr(obj, name)(*a, **k)))
    except Exception as exc:  # the exception class is part of the contract
        return ("err", type(exc).__name__)


def _groups(gs):
    return [(g.id, g.start, g.length, g.free, g.owner, g.active, g.filled) for g in gs]


def pool_fuzz(seed, be, steps=300):
    rnd = random.Random(seed)
    total = rnd.choice([16, 64, 200, 512])
    cfg = PoolConfig(total_blocks=total, initial_group_blocks=rnd.randint(1, min(60, total)),
                     rng_seed=rnd.randint(0, 2**40),
                     victim_policy=rnd.choice(["random", "lowest_priority"]))
    a, b = BlockGroupPool(cfg), native_ctrl.NativeBlockGroupPool(cfg, backend=backend(be))
    ranks = {}
    a.rank_of = b.rank_of = (lambda r: ranks.get(r, 10**6)) if rnd.random() < 0.8 else None
    reqs = list(range(rnd.randint(2, 12)))
    seen = set()
    for step in range(steps):
        op = rnd.random()
        r = rnd.choice(reqs)
        if rnd.random() < 0.1:
            ranks[r] = rnd.randint(0, 20)
        kw = {}
        if op < 0.35:
            name = "allocate"
            args = (r, rnd.randint(0 if rnd.random() < 0.02 else 1, max(1, total // 4)),
                    rnd.choice([None, rnd.randint(1, total)]), rnd.random() < 0.8)
        elif op < 0.45:
            gs = a.owned_groups(r)
            if not gs:
                continue
            name, args = "free_group", (rnd.choice(gs).id,)
        elif op < 0.5:
            name, args = "free_request", (r,)
        elif op < 0.6:
            gs = a.owned_groups(r)
            if not gs:
                continue
            g = rnd.choice(gs)
            name, args = "shrink_group", (g.id, rnd.randint(0, g.length + 1))
        elif op < 0.75:
            name = "set_request_fill"
            args = (r, rnd.randint(0, a.owned_blocks(r) + (1 if rnd.random() < 0.1 else 0)))
        elif op < 0.85:
            name, args = "allocate_at", (r, rnd.randint(0, total), rnd.randint(0, 20))
        elif op < 0.93:
            name, args, kw = "reclaim_from_victim", (rnd.randint(0, 12),), {"for_request": r}
        elif op < 0.96:
            name, args = "record_transfer", (rnd.randint(1, 40),)
        else:
            name, args = "free_group", (rnd.randint(0, 50),)
        ra, rb = _call(a, name, *args, **kw), _call(b, name, *args, **kw)
        assert ra == rb, (seed, step, name, args, ra, rb)
        seen.add((name, ra[0] if ra[0] == "ok" else ra[1]))
        if name == "allocate" and ra[0] == "ok" and ra[1][1]:
            seen.add(("allocate", "carved"))
        assert a.dump() == b.dump(), (seed, step, name)
        assert (a.free_blocks, a.used_blocks) == (b.free_blocks, b.used_blocks)
        x = rnd.choice(reqs)
        assert _groups(a.owned_groups(x)) == _groups(b.owned_groups(x))
        assert a.reclaimable_blocks(x) == b.reclaimable_blocks(x)
        assert a.reclaimable_blocks() == b.reclaimable_blocks()
        assert _groups(a.free_groups()) == _groups(b.free_groups())
        assert _call(a, "validate") == _call(b, "validate")
    assert a.granularity_stats() == b.granularity_stats()
    return seen


def _table(rnd, n):
    out, pos, left = [], rnd.randint(0, 1000), n
    while left > 0:
        k = rnd.randint(1, left)
        out.append((pos, k))
        pos += k + rnd.randint(0, 50)
        left -= k
    return out


def _copies(s):
    return {r: ([(x.block_lo, x.block_hi, x.group_id, x.valid) for x in s.copies[r].segments],
                s.copies[r].prealloc, s.copies[r].saved_tokens) for r in s.copies}


def store_fuzz(seed, be, steps=250):
    rnd = random.Random(seed)
    total = rnd.choice([32, 100, 256, 1024])
    kw = dict(reuse_enabled=rnd.random() < 0.8, prealloc_min_blocks=8, prealloc_max_blocks=256,
              release_on_swap_in=rnd.random() < 0.2, block_size_tokens=16)
    a = CpuStore(total, **kw)
    b = native_ctrl.NativeCpuStore(total, backend=backend(be), **kw)
    if rnd.random() < 0.2:
        a.refresh_dirty_tail = b.refresh_dirty_tail = False
    reqs = list(range(rnd.randint(2, 10)))
    fp = {r: 0 for r in reqs}
    seen = set()
    for step in range(steps):
        r = rnd.choice(reqs)
        op = rnd.random()
        if op < 0.1:
            rk = {x: rnd.randint(0, 10) for x in rnd.sample(reqs, rnd.randint(1, len(reqs)))}
            a.update_ranks(rk)
            b.update_ranks(rk)
            continue
        if op < 0.45:
            fp[r] = max(1, fp[r] + rnd.randint(-3, total // 6))
            name = "plan_swap_out"
            args = (r, fp[r], _table(rnd, fp[r]), rnd.choice([None, fp[r] * 16 - rnd.randint(0, 15)]))
        elif op < 0.6:
            c = a.copy_of(r)
            n = c.covered_blocks if c is not None and c.segments else rnd.randint(1, total)
            name, args = "plan_swap_in", (r, _table(rnd, n))
        elif op < 0.68:
            c = a.copy_of(r)
            n = c.valid_prefix_blocks() if c else 0
            name, args = "plan_swap_in_prefix", (r, _table(rnd, n) if n else [])
        elif op < 0.76:
            name, args = "evict_for", (rnd.randint(-1, 10), rnd.randint(0, total // 2))
        elif op < 0.86:
            name, args = "preallocate_increment", (r, rnd.randint(0, 40))
        elif op < 0.93:
            name, args = "release", (r,)
        else:
            rank = rnd.randint(0, 10)
            a.set_rank(r, rank)
            b.set_rank(r, rank)
            continue
        ra, rb = _call(a, name, *args), _call(b, name, *args)
        assert ra == rb, (seed, step, name, args, ra, rb)
        seen.add((name, ra[0] if ra[0] == "ok" else ra[1]))
        assert a.dump() == b.dump(), (seed, step, name)
        assert _copies(a) == _copies(b), (seed, step, name)
        assert dict(a.ranks) == dict(b.ranks)
        assert (a.peak_used_blocks, a.refreshed_blocks) == (b.peak_used_blocks, b.refreshed_blocks)
        b.pool.validate()
    return seen


@pytest.mark.parametrize("be", BACKENDS)
def test_pool_matches_python_control_plane_fuzz(be):
    seen = set()
    for seed in range(60 if be == "ext" else 25):
        seen |= pool_fuzz(seed, be)
    # the fuzz reached every decision path, error paths included
    for key in [("allocate", "ok"), ("allocate", "carved"), ("allocate", "OutOfMemoryError"),
                ("reclaim_from_victim", "ok"), ("reclaim_from_victim", "NoVictimError"),
                ("allocate_at", "ok"), ("shrink_group", "ok"), ("free_group", "PoolError"),
                ("set_request_fill", "PoolError")]:
        assert key in seen, key


@pytest.mark.parametrize("be", BACKENDS)
def test_cpu_store_matches_python_control_plane_fuzz(be):
    seen = set()
    for seed in range(40 if be == "ext" else 15):
        seen |= store_fuzz(seed, be)
    for key in [("plan_swap_out", "ok"), ("plan_swap_out", "CpuOutOfMemoryError"),
                ("plan_swap_in", "ok"), ("plan_swap_in", "ContaminatedCopyError"),
                ("plan_swap_in_prefix", "ok"), ("evict_for", "ok"),
                ("evict_for", "InsufficientVictimsError"), ("preallocate_increment", "ok")]:
        assert key in seen, key


# ---------------------------------------------------------------- goldens
def _native_mod(be):
    b = backend(be)
    return types.SimpleNamespace(
        PoolConfig=PoolConfig,
        BlockGroupPool=lambda cfg: native_ctrl.NativeBlockGroupPool(cfg, backend=b),
        CpuStore=lambda **kw: native_ctrl.NativeCpuStore(backend=b, **kw),
        ContaminatedCopyError=cpu_store.ContaminatedCopyError)


@pytest.mark.parametrize("be", BACKENDS)
def test_golden_op_sequences(be):
    mod = _native_mod(be)
    for args, want in tg.load("alloc.json")["cases"]:
        got = gg.alloc_sequence(mod, *args)
        assert got["final_dump"] == want["final_dump"]
        assert got["trail_sha256"] == want["trail_sha256"]
        assert list(got["granularity"] or []) == list(want["granularity"] or [])
    for args, want in tg.load("cpu_store.json")["cases"]:
        assert gg.cpu_store_sequence(mod, *args) == want


@pytest.mark.parametrize("name", sorted(tg.load("engine.json")))
def test_engine_goldens_on_native_control_plane(name, monkeypatch):
    """Every engine replay golden (report, event log, plan stream, pool
    dumps), with Engine.pool / Engine.store native."""
    monkeypatch.setattr(engine, "CONTROL_PLANE", "native")
    tg.test_engine_matches_reference(name, monkeypatch)


def test_engine_uses_the_native_classes():
    cfg = engine.EngineConfig(gpu_pool=PoolConfig(total_blocks=48, initial_group_blocks=20))
    eng = engine.Engine(cfg, [], control_plane="native")
    assert isinstance(eng.pool, native_ctrl.NativeBlockGroupPool)
    assert isinstance(eng.store, native_ctrl.NativeCpuStore)
    with pytest.raises(ValueError):
        engine.Engine(cfg, [], control_plane="bogus")


def test_errors_are_the_reference_classes():
    pool = native_ctrl.NativeBlockGroupPool(PoolConfig(total_blocks=32, initial_group_blocks=4))
    g = pool.allocate(1, 4).groups[0]
    pool.free_group(g.id)
    with pytest.raises(alloc.PoolError):
        pool.free_group(g.id)
    with pytest.raises(alloc.OutOfMemoryError):
        pool.allocate(2, 33)
    with pytest.raises(ValueError):
        pool.allocate(2, 0)
    with pytest.raises(alloc.NoVictimError):
        pool.reclaim_from_victim(4, for_request=3)
    store = native_ctrl.NativeCpuStore(total_blocks=16)
    with pytest.raises(cpu_store.ContaminatedCopyError):
        store.plan_swap_in(7, [(0, 4)])
    store.set_rank(1, 0)
    store.plan_swap_out(1, 16, [(0, 16)])
    with pytest.raises(cpu_store.CpuOutOfMemoryError):
        store.plan_swap_out(2, 4, [(0, 4)])  # rank 0 copy cannot be evicted for rank 0


def test_rank_callback_errors_propagate():
    pool = native_ctrl.NativeBlockGroupPool(PoolConfig(total_blocks=16, initial_group_blocks=16,
                                                       victim_policy="lowest_priority"))
    pool.allocate(1, 2, expected_total=16)  # one active group with a 14-block tail

    def boom(req):
        raise RuntimeError("rank lookup failed")

    pool.rank_of = boom
    with pytest.raises(RuntimeError, match="rank lookup failed"):
        pool.reclaim_from_victim(4, for_request=2)


REF_TESTS = Path("/root/reference/pkg/tests")
SHIM = '''
import importlib, sys
sys.path.insert(0, {root!r})
import paper_2411_18424_b200 as pkg
sys.modules["kvswitch"] = pkg
for m in {mods!r}:
    sys.modules["kvswitch." + m] = importlib.import_module("paper_2411_18424_b200." + m)
from paper_2411_18424_b200 import alloc, cpu_store, engine, native_ctrl
alloc.BlockGroupPool = native_ctrl.NativeBlockGroupPool
cpu_store.CpuStore = native_ctrl.NativeCpuStore
engine.CONTROL_PLANE = "native"
'''
CHECK = '''
from kvswitch.alloc import BlockGroupPool, PoolConfig
from kvswitch.cpu_store import CpuStore
from kvswitch.engine import Engine, EngineConfig
from paper_2411_18424_b200 import native_ctrl


def test_suite_runs_on_the_native_classes():
    assert BlockGroupPool is native_ctrl.NativeBlockGroupPool
    assert CpuStore is native_ctrl.NativeCpuStore
    eng = Engine(EngineConfig(gpu_pool=PoolConfig(total_blocks=48, initial_group_blocks=20)), [])
    assert isinstance(eng.pool, native_ctrl.NativeBlockGroupPool)
'''


@pytest.mark.skipif(not REF_TESTS.is_dir(), reason="reference not mounted")
def test_reference_suite_passes_on_native_control_plane(tmp_path):
    files = ["alloc", "core", "costmodel", "cpu_store", "engine", "scheduler", "swap",
             "workload"]
    (tmp_path / "conftest.py").write_text(SHIM.format(root=str(ROOT), mods=files))
    for f in files:
        src = REF_TESTS / f"test_{f}.py"
        (tmp_path / src.name).write_text(src.read_text())
    (tmp_path / "test_zz_native.py").write_text(CHECK)
    res = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                          str(tmp_path)], capture_output=True, text=True, cwd=tmp_path,
                         timeout=900)
    tail = res.stdout[-3000:]
    assert res.returncode == 0, tail
    assert "124 passed" in tail, tail
