"""Run documents and trace I/O (the callers' plumbing around the swap path)."""

import pytest

from paper_2411_18424_b200 import config as mconfig
from paper_2411_18424_b200.geometry import LLAMA3_8B, LLAMA3_70B, QWEN25_32B
from paper_2411_18424_b200.workload import WorkloadConfig, generate, ingest, write_trace


def test_build_fans_out_the_seed():
    eng, wl, full = mconfig.build({"seed": 7, "ablation": "baseline",
                                   "gpu_pool": {"total_blocks": 300}})
    assert eng.gpu_pool.rng_seed == 7 and eng.trace.seed == 7 and wl.seed == 7
    assert eng.ablation == "baseline" and eng.gpu_pool.total_blocks == 300
    assert full["workload"]["max_context_tokens"] == 3072  # reference default document


def test_unknown_keys_and_bad_values_rejected():
    with pytest.raises(mconfig.ConfigError):
        mconfig.build({"gpu_pool": {"blocks": 3}})
    with pytest.raises(mconfig.ConfigError):
        mconfig.build({"ablation": "turbo"})
    with pytest.raises(mconfig.ConfigError):
        mconfig.build({"trace": {"pattern": "zipf"}})


def test_trace_round_trip(tmp_path):
    convs = generate(WorkloadConfig(num_conversations=9, seed=3, max_context_tokens=2048))
    path = tmp_path / "t.jsonl"
    write_trace(convs, path)
    back = ingest(path)
    assert [(c.id, c.turns, c.arrival, c.think_time) for c in back] == \
        [(c.id, c.turns, c.arrival, c.think_time) for c in convs]
    path.write_text('{"id": 1}\n')
    with pytest.raises(ValueError, match="line 1"):
        ingest(path)


def test_geometry_block_bytes_match_baseline_table():
    # per-rank all-layer block bytes at 16 tokens, fp16, d=128, 8 KV heads
    assert LLAMA3_8B.block_bytes == 2 << 20 and LLAMA3_8B.plane_chunk_bytes == 64 << 10
    assert [QWEN25_32B.with_tp(t).block_bytes for t in (2, 4, 8)] == [2 << 20, 1 << 20, 512 << 10]
    assert LLAMA3_70B.with_tp(8).block_bytes == 655360
    assert LLAMA3_70B.with_tp(8).plane_chunk_bytes == 8192
    assert LLAMA3_8B.block_spec().bytes_per_block == LLAMA3_8B.block_bytes
    with pytest.raises(ValueError):
        LLAMA3_8B.with_tp(3)
