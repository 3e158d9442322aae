"""The oracle itself: numpy restatement vs C restatement, TransferOp
semantics (cpu_store.py:73-120), split-single equivalence (swap.py:170-179),
and pinned KV-pattern vectors."""

import hashlib

import numpy as np
import pytest

from oracle import bytes_oracle as orc
from oracle import c_oracle


def test_kv_pattern_pinned():
    a = orc.kv_pattern(7, 3, 5, 64)
    assert a.shape == (3, 5, 64)
    # golden digest: changes to the hash would silently change every fixture
    assert hashlib.sha256(a.tobytes()).hexdigest()[:16] == PINNED_PATTERN
    b = orc.kv_pattern(8, 3, 5, 64)
    assert not np.array_equal(a, b)
    # every (plane, block) chunk distinct
    chunks = {a[p, k].tobytes() for p in range(3) for k in range(5)}
    assert len(chunks) == 15


PINNED_PATTERN = "2e425f7d885ac284"


def test_pattern_words_pinned():
    assert orc.kv_pattern(1, 1, 1, 16).view(np.uint32)[0, 0].tolist() == PINNED_WORDS


PINNED_WORDS = [301794027, 2980047484, 2117216093, 2789948889]


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_numpy_and_c_oracles_agree(seed):
    rng = np.random.default_rng(seed)
    P, G, C, chunk = 4, 64, 48, 272
    planes = orc.kv_pattern(seed, P, G, chunk)
    gtab = orc.random_block_table(rng, 30, G)
    ctab = orc.random_block_table(rng, 30, C)
    ops = orc.table_to_ops(gtab, ctab)
    h1 = np.zeros((C, P * chunk), np.uint8)
    h2 = np.zeros((C, P * chunk), np.uint8)
    orc.apply_plan("out", planes.copy(), h1, ops)
    c_oracle.apply_plan_arrays("out", planes.copy(), h2, ops, nthreads=3)
    assert np.array_equal(h1, h2)
    p1 = np.zeros_like(planes)
    p2 = np.zeros_like(planes)
    orc.apply_plan("in", p1, h1, ops)
    c_oracle.apply_plan_arrays("in", p2, h1, ops, nthreads=2)
    assert np.array_equal(p1, p2)
    for k in range(30):
        assert np.array_equal(p1[:, gtab[k]], planes[:, gtab[k]])


def test_split_single_moves_identical_bytes():
    rng = np.random.default_rng(4)
    planes = orc.kv_pattern(4, 2, 40, 32)
    ops = orc.random_runs(rng, 24, 6, 40, 40)
    a = np.zeros((40, 64), np.uint8)
    b = np.zeros((40, 64), np.uint8)
    orc.apply_plan("out", planes, a, ops)
    orc.apply_plan("out", planes, b, orc.split_single(ops))
    assert np.array_equal(a, b)
    assert orc.split_single(ops).shape[0] == 24


def test_table_to_ops_is_pair_extents_rule():
    # breaks wherever either side loses contiguity
    ops = orc.table_to_ops([5, 6, 7, 20, 21], [0, 1, 9, 10, 11])
    assert ops.tolist() == [[2, 5, 0], [1, 7, 9], [2, 20, 10]]
    assert orc.block_pairs(ops).tolist() == [[5, 0], [6, 1], [7, 9], [20, 10], [21, 11]]


def test_apply_plan_rejects_bad_ops():
    planes = np.zeros((1, 4, 16), np.uint8)
    host = np.zeros((4, 16), np.uint8)
    with pytest.raises(IndexError):
        orc.apply_plan("out", planes, host, [(2, 3, 0)])
    with pytest.raises(IndexError):
        orc.apply_plan("out", planes, host, [(0, 0, 0)])
    with pytest.raises(ValueError):
        orc.apply_plan("up", planes, host, [(1, 0, 0)])


def test_random_runs_are_disjoint():
    rng = np.random.default_rng(0)
    ops = orc.random_runs(rng, 100, 7, 300, 200)
    assert ops[:, 0].sum() == 100
    g = np.concatenate([np.arange(gs, gs + b) for b, gs, _ in ops])
    c = np.concatenate([np.arange(cs, cs + b) for b, _, cs in ops])
    assert len(set(g)) == 100 and len(set(c)) == 100


def test_synthetic_generators_agree_with_the_oracle_restatement():
    """bench.py / tools build plans with paper_2411_18424_b200.synthetic; the
    pairing rule must be the oracle's (_pair_extents, cpu_store.py:95-120)."""
    from paper_2411_18424_b200 import synthetic as syn

    for seed in range(20):
        rng = np.random.default_rng(seed)
        g = syn.random_block_table(rng, 300, 1000)
        c = syn.random_block_table(rng, 300, 1000)
        runs = np.concatenate([np.arange(s, s + 40) for s in (5, 500, 300)])
        g2, c2 = np.concatenate([g, runs]), np.concatenate([c, runs + 3])
        np.testing.assert_array_equal(syn.pair_tables(g2, c2), orc.table_to_ops(g2, c2))
        a = syn.random_runs(np.random.default_rng(seed), 512, 16, 2048, 2048)
        b = orc.random_runs(np.random.default_rng(seed), 512, 16, 2048, 2048)
        np.testing.assert_array_equal(a, b)  # same seeded layout as the oracle's generator
