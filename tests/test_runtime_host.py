"""Host-side logic of the runtime (no GPU): token spans -> KV-write segments."""

import numpy as np
import pytest

from paper_2411_18424_b200.runtime import token_segments


def expand(segs, T):
    """segments -> {(req, token): (physical block, slot)}"""
    out = {}
    for req, lo, hi, phys in segs.tolist():
        for t in range(lo, hi):
            out[(req, t)] = (phys + t // T - lo // T, t % T)
    return out


def brute(spans, tables, T):
    out = {}
    for req, lo, hi in spans:
        flat = [b for s, n in tables[req] for b in range(s, s + n)]
        for t in range(lo, hi):
            out[(req, t)] = (flat[t // T], t % T)
    return out


@pytest.mark.parametrize("seed", range(20))
def test_segments_match_block_table(seed):
    rng = np.random.default_rng(seed)
    T = 16
    tables, spans = {}, []
    for req in range(6):
        n_ext = int(rng.integers(1, 6))
        starts = rng.choice(1000, size=n_ext, replace=False) * 8
        tables[req] = [(int(s), int(rng.integers(1, 8))) for s in starts]
        cap = sum(n for _, n in tables[req]) * T
        lo = int(rng.integers(0, cap))
        hi = int(rng.integers(lo, cap + 1))
        spans.append((req, lo, hi))
    segs = token_segments(spans, tables.__getitem__, T)
    assert expand(segs, T) == brute(spans, tables, T)
    # each segment stays inside one physically contiguous extent
    for req, lo, hi, phys in segs.tolist():
        last = phys + (hi - 1) // T - lo // T
        assert any(s <= phys and last < s + n for s, n in tables[req])


def test_empty_and_overflowing_spans():
    tables = {0: [(10, 2)]}
    assert token_segments([(0, 5, 5)], tables.__getitem__, 16).shape == (0, 4)
    with pytest.raises(IndexError):
        token_segments([(0, 0, 33)], tables.__getitem__, 16)


def test_swap_rate_summary_splits_alone_duplex_and_plan_size():
    from paper_2411_18424_b200.runtime import swap_rate_summary

    mib = 1 << 20
    iv = {  # (start ms, end ms, bytes) on the device timeline
        "out": [(0.0, 1.0, 50 * mib), (10.0, 12.0, 100 * mib)],
        "in": [(2.0, 3.0, 40 * mib),          # alone
               (10.0, 11.0, 36 * mib),        # fully inside the second swap-out
               (20.0, 20.1, 4 * mib)],        # small plan, alone
    }
    r = swap_rate_summary(iv)
    assert r["in"]["transfers"] == 3 and r["in"]["transfers_alone"] == 2
    assert r["in"]["transfers_overlapping"] == 1
    assert r["in"]["gbs_overlapping_other_direction"] == round(36 * mib / 1e-3 / 1e9, 2)
    assert abs(r["in"]["gbs_plans_lt_32mib"] - 4 * mib / 0.1e-3 / 1e9) < 0.01
    assert r["out"]["transfers_alone"] == 1  # the first swap-out ran alone
    assert r["out"]["gbs_while_busy"] == round(150 * mib / 3e-3 / 1e9, 2)


def test_pcie_switch_groups_from_the_pcie_only_topology_matrix():
    from paper_2411_18424_b200.dataplane import pcie_switch_groups

    txt = ("\tGPU0\tGPU1\tGPU2\tGPU3\tNIC0\tCPU Affinity\tNUMA Affinity\tGPU NUMA ID\n"
           "GPU0\t X \tPIX\tNODE\tSYS\tPXB\t0-55\t0\t\tN/A\n"
           "GPU1\tPIX\t X \tNODE\tSYS\tPXB\t0-55\t0\t\tN/A\n"
           "GPU2\tNODE\tNODE\t X \tSYS\tNODE\t0-55\t0\t\tN/A\n"
           "GPU3\tSYS\tSYS\tSYS\t X \tSYS\t56-111\t1\t\tN/A\n")
    got = pcie_switch_groups(4, txt)
    assert got["groups"] == [[0, 1], [2], [3]]  # GPU0/1 share a switch uplink
    assert got["matrix"]["0-2"] == "NODE"
    assert pcie_switch_groups(2, txt)["groups"] == [[0, 1]]
    assert pcie_switch_groups(2, "no matrix here") == {}
