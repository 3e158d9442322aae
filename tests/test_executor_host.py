"""Host-side hazard logic of the StreamExecutor (no GPU): which TransferOps
of an in-flight transfer a new transfer or compute must wait for."""

import numpy as np
import pytest

from paper_2411_18424_b200.swap import DUPLEX_POLICIES, _hit_ops, _overlaps


def brute_hits(extents, per_op):
    hit = []
    for i, (s1, n1) in enumerate(per_op):
        blocks = set(range(s1, s1 + n1))
        if any(blocks & set(range(s0, s0 + n0)) for s0, n0 in extents):
            hit.append(i)
    return hit


@pytest.mark.parametrize("seed", range(30))
def test_hit_ops_is_half_open_interval_intersection(seed):
    rng = np.random.default_rng(seed)
    per_op = [(int(rng.integers(0, 200)), int(rng.integers(1, 12))) for _ in range(8)]
    extents = [(int(rng.integers(0, 200)), int(rng.integers(1, 12)))
               for _ in range(int(rng.integers(0, 4)))]
    assert _hit_ops(extents, per_op) == brute_hits(extents, per_op)
    assert _overlaps(extents, per_op) == bool(brute_hits(extents, per_op))


def test_adjacent_extents_do_not_conflict():
    # [10, 14) and [14, 20) touch but share no block (swap.py:236-245 half-open rule)
    assert _hit_ops([(10, 4)], [(14, 6)]) == []
    assert _hit_ops([(10, 5)], [(14, 6)]) == [0]


def test_duplex_policies_are_well_formed():
    for name, pol in DUPLEX_POLICIES.items():
        path = pol.get("path", "lsu")
        assert path in ("lsu", "bulk"), name
        for d in ("out", "in"):
            ctas, threads, pace = pol[d]
            assert ctas >= 1 and threads % 32 == 0, name
            assert (32 <= threads <= 1024) if path == "lsu" else threads == 0, name
            assert pace >= 0.0
        assert pol["budget"] >= 0.0
        for d, eng in pol.get("engine", {}).items():
            assert d in ("out", "in") and eng in ("kernel", "ce_per_block", "ce_per_run",
                                                  "ce_staged"), name
        for d, gbps in pol.get("share", {}).items():
            assert d in ("out", "in") and 0.0 < gbps <= pol["budget"], name
    # serving: swap-out paced below the link, swap-in bounded by reads in flight
    lat = DUPLEX_POLICIES["latency"]
    assert 0 < lat["out"][2] < 63.0
    assert lat["in"][2] == 0.0 and lat["in"][0] * lat["in"][1] // 32 * 4096 <= 512 * 1024
    # the live traces' policy (graph-launched decode): swap-in paced just under
    # the link and bounded by reads in flight, swap-out paced below the link,
    # swap-in keeps a reserved share of the shared budget while both run;
    # serving_link is the same with swap-in at the link rate
    srv = DUPLEX_POLICIES["serving"]
    assert 40.0 <= srv["in"][2] < 51.4 and 0 < srv["out"][2] < 63.0
    assert srv["in"][0] * srv["in"][1] // 32 * 4096 <= 512 * 1024
    assert 0 < srv["share"]["in"] < srv["budget"]
    link = DUPLEX_POLICIES["serving_link"]
    assert link["in"][2] == 0.0 and {k: v for k, v in link.items() if k != "in"} == \
        {k: v for k, v in srv.items() if k != "in"}
    # stream-launched decode: both directions paced below the link, under the budget
    sp = DUPLEX_POLICIES["serving_paced"]
    assert 0 < sp["out"][2] <= sp["in"][2] < 63.0
    assert sp["out"][2] + sp["in"][2] <= sp["budget"]
