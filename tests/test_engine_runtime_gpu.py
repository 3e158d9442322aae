"""End-to-end byte integrity of the swap path on the GPU: the engine (replay
mode, decisions bit-exact with the reference) drives real swaps through
libkvswap while the compute stream writes every produced token's KV; every
swap-in is read back and compared with the tokens' deterministic pattern."""

import json
from pathlib import Path

import pytest

from paper_2411_18424_b200 import config as mconfig
from paper_2411_18424_b200.alloc import PoolConfig
from paper_2411_18424_b200.engine import Engine, EngineConfig
from paper_2411_18424_b200.geometry import KVGeometry
from paper_2411_18424_b200.scheduler import PriorityTrace
from paper_2411_18424_b200.workload import Conversation, WorkloadConfig, generate

pytestmark = pytest.mark.gpu

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "engine.json").read_text())
TINY = KVGeometry("tiny-kv", num_layers=2, num_kv_heads=2, head_dim=8)  # 1 KiB chunks


def _runtime(cfg, **kw):
    from paper_2411_18424_b200.runtime import Runtime
    cpu = min(cfg.cpu_pool_blocks, 8192)
    return Runtime(TINY, cfg.gpu_pool.total_blocks, cpu, verify=True, **kw)


def _cfg_small(**over):
    base = dict(gpu_pool=PoolConfig(total_blocks=48, initial_group_blocks=20),
                trace=PriorityTrace(pattern="random", frequency=0.2, seed=1), ablation="full",
                cpu_pool_blocks=4096)
    base.update(over)
    return EngineConfig(**base)


def duel():
    return [Conversation(0, [(320, 320)], 0, 0), Conversation(1, [(320, 320)], 1000, 0)]


@pytest.mark.parametrize("copy_impl", ["kernel", "ce_per_block", "ce_staged"])
def test_duel_bytes_and_golden_decisions(cuda_ok, copy_impl):
    cfg = _cfg_small()
    rt = _runtime(cfg, copy_impl=copy_impl)
    eng = Engine(cfg, duel(), runtime=rt)
    eng.check_invariants = True
    rep = json.loads(eng.run().to_json())
    rt.synchronize()
    want = dict(GOLD["duel_full"]["report"])
    want["peak_cpu_blocks"] = rep["peak_cpu_blocks"]  # smaller host pool than the golden's
    assert rep == want  # real bytes do not perturb replay decisions
    assert rt.verified > 0 and rt.stats()["bytes_out"] > 0
    rt.close()


@pytest.mark.parametrize("ablation", ["baseline", "blockgroup", "blockgroup_reuse", "full"])
def test_multiturn_trace_integrity(cuda_ok, ablation):
    convs = generate(WorkloadConfig(num_conversations=12, seed=5, max_context_tokens=2048))
    cfg = EngineConfig(gpu_pool=PoolConfig(total_blocks=256, initial_group_blocks=60),
                       trace=PriorityTrace(pattern="markov", frequency=0.04, seed=2),
                       ablation=ablation, cpu_pool_blocks=4096)
    rt = _runtime(cfg)
    eng = Engine(cfg, convs, runtime=rt)
    rep = eng.run()
    rt.synchronize()
    assert rep.total_tokens == rep.expected_tokens
    assert rt.verified > 0
    if ablation in ("blockgroup_reuse", "full"):
        assert eng.store.refreshed_blocks > 0  # dirty tails were re-sent
    rt.close()


def test_pressure_trace_with_contamination(cuda_ok):
    cfg, wl, _ = mconfig.build({"ablation": "full", "gpu_pool": {"total_blocks": 256},
                                "cpu_pool": {"total_blocks": 600},
                                "workload": {"arrival_rate_per_s": 3.0, "num_conversations": 30},
                                "trace": {"pattern": "random", "frequency": 0.04}})
    rt = _runtime(cfg)
    eng = Engine(cfg, generate(wl), runtime=rt)
    rep = eng.run()
    rt.synchronize()
    assert rep.total_tokens == rep.expected_tokens
    assert rt.verified > 0
    rt.close()


def test_without_dirty_tail_refresh_bytes_go_stale(cuda_ok):
    """SURVEY §0 finding 3: the reference's reuse accounting alone restores
    stale tail blocks; the refresh op is what makes the bytes sound."""
    from paper_2411_18424_b200.runtime import KVIntegrityError

    convs = generate(WorkloadConfig(num_conversations=12, seed=5, max_context_tokens=2048))
    cfg = EngineConfig(gpu_pool=PoolConfig(total_blocks=256, initial_group_blocks=60),
                       trace=PriorityTrace(pattern="markov", frequency=0.04, seed=2),
                       ablation="full", cpu_pool_blocks=4096)
    rt = _runtime(cfg)
    eng = Engine(cfg, convs, runtime=rt)
    eng.store.refresh_dirty_tail = False
    with pytest.raises(KVIntegrityError):
        eng.run()
    rt.close()


def test_live_engine_bytes_and_latency(cuda_ok):
    """Live mode: real clock, event-driven swap completion, real decode kernel.
    Decisions diverge from replay by design; bytes must still be exact."""
    from paper_2411_18424_b200.live import DecodeEmulator, LiveEngine, b200_transfer_params

    convs = generate(WorkloadConfig(num_conversations=10, seed=5, max_context_tokens=2048,
                                    arrival_rate_per_s=20.0, think_time_mean_s=0.05))
    cfg = EngineConfig(gpu_pool=PoolConfig(total_blocks=128, initial_group_blocks=40),
                       trace=PriorityTrace(pattern="random", frequency=0.04, seed=2),
                       ablation="full", cpu_pool_blocks=4096, transfer=b200_transfer_params())
    rt = _runtime(cfg, timing=True)
    dec = DecodeEmulator("cuda:0", weight_bytes=1 << 30)
    eng = LiveEngine(cfg, convs, rt, dec)
    rep = eng.run()
    lat = eng.latency_summary()
    assert rep.total_tokens == rep.expected_tokens
    assert rep.swap_out_blocks > 0 and rt.verified > 0
    assert lat["ttft_p99_ms"] is not None and lat["tbt_p99_ms"] > 0
    assert dec.bytes_per_us > 1e6  # > 1 TB/s calibrated weight streaming
    assert rt.kv_bytes_read > 0 and rt.kv_errors() == 0  # decode read every resident KV byte
    rt.close()


@pytest.mark.parametrize("geo_name", ["tiny", "llama3-8b", "llama3-70b-tp8"])
def test_kv_token_kernel_matches_torch_pattern(cuda_ok, geo_name):
    """kvs_kv_tokens (write + check) against the plain torch restatement."""
    import numpy as np
    import torch

    from paper_2411_18424_b200.geometry import PRESETS
    from paper_2411_18424_b200.runtime import Runtime, token_segments

    geo = (TINY if geo_name == "tiny" else PRESETS["llama3-70b"].with_tp(8)
           if geo_name == "llama3-70b-tp8" else PRESETS[geo_name])
    G = 64
    rt = Runtime(geo, G, 8, verify=True)
    rt.cache.planes.fill_(0)
    T = geo.block_tokens
    tables = {3: [(40, 3), (5, 2)], 9: [(20, 4)], 123456: [(60, 4)]}
    spans = [(3, 7, 70), (9, 0, 64), (123456, 17, 18)]
    segs = token_segments(spans, tables.__getitem__, T)
    s = rt.executor.compute
    rt.dataplane.kv_tokens(0, segs, stream=s)
    s.synchronize()
    want = torch.zeros_like(rt._slots)
    for req, lo, hi in spans:
        flat = [b for st, n in tables[req] for b in range(st, st + n)]
        t = torch.arange(lo, hi, device=want.device)
        p = torch.tensor([flat[x // T] for x in range(lo, hi)], device=want.device)
        r = torch.full_like(t, req)
        want[:, p, :, t % T, :] = rt._pattern(r, t)
    assert torch.equal(rt._slots, want)
    # check mode: exact -> 0; one flipped word -> counted
    rt._mismatch.zero_()
    rt.dataplane.kv_tokens(1, segs, stream=s, mismatch_ptr=rt._mismatch.data_ptr())
    s.synchronize()
    assert int(rt._mismatch.item()) == 0
    rt._slots[1, 41, 1, 3, 0] ^= 1  # req 3, token 19 -> block 41 slot 3, plane 1, V
    torch.cuda.synchronize()
    rt._mismatch.zero_()
    rt.dataplane.kv_tokens(1, segs, stream=s, mismatch_ptr=rt._mismatch.data_ptr())
    s.synchronize()
    assert int(rt._mismatch.item()) == 1
    with pytest.raises(IndexError):
        rt.dataplane.kv_tokens(0, np.array([[0, 0, 32, G - 1]]), stream=s)
    rt.close()


def test_live_engine_layered_admission_bytes(cuda_ok):
    """Layered admission: resumed requests join decode layer by layer (plane
    flags); every joined request's KV is verified after its layers landed."""
    from paper_2411_18424_b200.live import DecodeEmulator, LiveEngine, b200_transfer_params

    convs = generate(WorkloadConfig(num_conversations=10, seed=5, max_context_tokens=2048,
                                    arrival_rate_per_s=20.0, think_time_mean_s=0.05))
    cfg = EngineConfig(gpu_pool=PoolConfig(total_blocks=128, initial_group_blocks=40),
                       trace=PriorityTrace(pattern="random", frequency=0.04, seed=2),
                       ablation="full", cpu_pool_blocks=4096, transfer=b200_transfer_params())
    rt = _runtime(cfg, timing=True, layered_swap_in=True)
    dec = DecodeEmulator("cuda:0", weight_bytes=1 << 30)
    eng = LiveEngine(cfg, convs, rt, dec, layered=True)
    rep = eng.run()
    lat = eng.latency_summary()
    assert rep.total_tokens == rep.expected_tokens
    assert eng.layered_joins > 0 and rt.verified > 0
    assert lat["layered_joins"] == eng.layered_joins
    assert rt.kv_bytes_read > 0 and rt.kv_errors() == 0
    rt.close()


def test_live_attention_reads_catch_corruption(cuda_ok):
    """The attention stand-in checks every resident KV byte it reads: a byte
    flipped in a running request's block fails the run."""
    import torch

    from paper_2411_18424_b200.live import DecodeEmulator, LiveEngine, b200_transfer_params
    from paper_2411_18424_b200.runtime import KVIntegrityError

    convs = [Conversation(0, [(320, 200)], 0, 0)]
    cfg = EngineConfig(gpu_pool=PoolConfig(total_blocks=64, initial_group_blocks=40),
                       trace=PriorityTrace(pattern="random", frequency=0.04, seed=2),
                       ablation="full", cpu_pool_blocks=256, transfer=b200_transfer_params())
    rt = _runtime(cfg)
    dec = DecodeEmulator("cuda:0", weight_bytes=1 << 30)
    eng = LiveEngine(cfg, convs, rt, dec)
    writes = {"n": 0}
    orig = rt.write

    def corrupting_write(engine, spans):
        orig(engine, spans)
        writes["n"] += 1
        if writes["n"] == 20:  # after a few decode steps: flip one word of token 3's K row
            start, _ = engine._gpu_extents(0)[0]
            with torch.cuda.stream(rt.executor.compute):
                rt._slots[0, start, 0, 3, 0] ^= 1
    rt.write = corrupting_write
    with pytest.raises(KVIntegrityError):
        eng.run()
    rt.close()


def test_live_engine_flag_ring_wraps(cuda_ok):
    """A tiny completion-word ring wraps many times during a live run: slots
    are only recycled once the transfer that owned them has landed, so every
    op / plane wait still sees its own transfer (bytes verified)."""
    from paper_2411_18424_b200.live import DecodeEmulator, LiveEngine, b200_transfer_params

    convs = generate(WorkloadConfig(num_conversations=10, seed=5, max_context_tokens=2048,
                                    arrival_rate_per_s=20.0, think_time_mean_s=0.05))
    cfg = EngineConfig(gpu_pool=PoolConfig(total_blocks=128, initial_group_blocks=40),
                       trace=PriorityTrace(pattern="random", frequency=0.04, seed=2),
                       ablation="full", cpu_pool_blocks=4096, transfer=b200_transfer_params())
    rt = _runtime(cfg, layered_swap_in=True, flag_ring=64)
    dec = DecodeEmulator("cuda:0", weight_bytes=1 << 30)
    eng = LiveEngine(cfg, convs, rt, dec, layered=True)
    rep = eng.run()
    assert rep.total_tokens == rep.expected_tokens and rt.verified > 0
    assert rt.executor._seq * 3 > 64  # many more completion words than ring slots
    assert rt.kv_errors() == 0
    rt.close()


def test_native_control_plane_drives_real_bytes(cuda_ok):
    """Engine(control_plane="native"): the C++ pool / store plan every swap of
    a multi-turn trace; decisions equal the Python control plane's and every
    swap-in is byte-verified."""
    convs = generate(WorkloadConfig(num_conversations=12, seed=5, max_context_tokens=2048))
    cfg = EngineConfig(gpu_pool=PoolConfig(total_blocks=256, initial_group_blocks=60),
                       trace=PriorityTrace(pattern="random", frequency=0.2, seed=2),
                       ablation="full", cpu_pool_blocks=2048)
    reports = {}
    for cp in ("python", "native"):
        rt = _runtime(cfg)
        eng = Engine(cfg, convs, runtime=rt, control_plane=cp)
        reports[cp] = json.loads(eng.run().to_json())
        rt.synchronize()
        assert rt.verified > 0
        rt.close()
    assert reports["native"] == reports["python"]


@pytest.mark.parametrize("n_segs", [31, 32, 33, 256, 257, 600])
def test_kv_token_kernel_size_classes(cuda_ok, n_segs):
    """kvs_kv_tokens across its parameter size classes (32 and 256 segments
    per launch, more in several launches): n one-token segments on distinct
    blocks written, checked exact, then one flipped word counted once."""
    import numpy as np
    import torch

    from paper_2411_18424_b200.runtime import Runtime

    G = 640
    rt = Runtime(TINY, G, 8, verify=True)
    rt.cache.planes.fill_(0)
    segs = np.array([[7 + i, i % TINY.block_tokens, i % TINY.block_tokens + 1, i]
                     for i in range(n_segs)], dtype=np.int64)
    s = rt.executor.compute
    rt.dataplane.kv_tokens(0, segs, stream=s)
    rt._mismatch.zero_()
    rt.dataplane.kv_tokens(1, segs, stream=s, mismatch_ptr=rt._mismatch.data_ptr())
    s.synchronize()
    assert int(rt._mismatch.item()) == 0
    # every segment's row landed: block i holds request 7+i's token
    assert int((rt.cache.planes[:, :n_segs] != 0).any(dim=-1).sum().item()) == \
        TINY.num_planes * n_segs
    last = n_segs - 1
    rt._slots[0, last, 0, last % TINY.block_tokens, 0] ^= 1
    torch.cuda.synchronize()
    rt._mismatch.zero_()
    rt.dataplane.kv_tokens(1, segs, stream=s, mismatch_ptr=rt._mismatch.data_ptr())
    s.synchronize()
    assert int(rt._mismatch.item()) == 1
    rt.close()
