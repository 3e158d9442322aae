"""VTC (Virtual Token Counter, Sheng et al. OSDI'24) — the fairness-aware
priority source of BASELINE config 3.

The reference has no VTC, so parity is pinned two ways:
  * the counter primitives are checked call for call against
    oracle/vtc_oracle.py's independent restatement of Alg. 2, including the
    paper's own continuous-batching setting, where VTC's fairness bound
    U = max(w_p L_input, w_q M) must hold for backlogged clients;
  * the engine's preemption / resume decisions under "vtc" are compared with
    the UNMODIFIED reference engine driven by the oracle's VTC
    (tests/golden/engine.json "vtc_*" cases in test_golden.py; a live
    differential over random configurations here, when the reference is
    present)."""

import json
import os
import random

import pytest

from oracle import vtc_oracle as vo
from paper_2411_18424_b200 import config as mconfig
from paper_2411_18424_b200.engine import Engine
from paper_2411_18424_b200.scheduler import (PriorityTrace, VirtualTokenCounters,
                                             apply_priority_update)
from paper_2411_18424_b200.workload import generate

VTC_TRACE = PriorityTrace(pattern="vtc", frequency=0.1)


class _ProductVTC:
    """The oracle server's calls, answered by the product's primitives."""

    def __init__(self, wp, wq):
        self.v = VirtualTokenCounters(wp, wq)

    def arrive(self, u, backlog):
        self.v.backlogged(u, [b for b in backlog if b != u])

    def depart(self, u):
        self.v.left(u)

    def serve(self, u, prompt=0, output=0):
        self.v.charge(u, prefill=prompt, decode=output)

    def counter(self, u):
        return self.v.get(u)

    def pick(self, cands):
        ranks = apply_priority_update(0, VTC_TRACE, list(cands), [], self.v.counters)
        return min(ranks, key=ranks.get)


def _requests(seed):
    r = random.Random(seed)
    reqs = []
    for u in range(r.randint(2, 6)):
        rate, t = r.choice([0.05, 0.2, 0.5, 1.0]), r.randint(0, 50)
        while t < 1200:
            reqs.append((t, u, r.randint(1, 256), r.randint(1, 128)))
            t += max(1, int(r.expovariate(rate)))
    return reqs, r.choice([512, 1024, 2048])


def test_vtc_ranks_least_counter_first_ties_by_id():
    ranks = apply_priority_update(3, VTC_TRACE, live=[7, 2, 9, 4], running=[2, 9],
                                  served={7: 50, 2: 10, 9: 10, 4: 0})
    assert ranks == {4: 0, 2: 1, 9: 2, 7: 3}
    # RNG-free: the epoch number and the running set do not matter
    assert apply_priority_update(99, VTC_TRACE, [7, 2, 9, 4], [],
                                 {7: 50, 2: 10, 9: 10, 4: 0}) == ranks
    assert apply_priority_update(1, VTC_TRACE, [5, 1], [], None) == {1: 0, 5: 1}


def test_counter_primitives_match_oracle_call_for_call():
    rng = random.Random(7)
    ours, ref = VirtualTokenCounters(1, 2), vo.VTC(1, 2)
    live: set = set()
    for _ in range(5000):
        u = rng.randrange(12)
        op = rng.random()
        if op < 0.25 and u not in live:
            ours.backlogged(u, sorted(live))
            ref.arrive(u, sorted(live))
            live.add(u)
        elif op < 0.4 and u in live:
            ours.left(u)
            ref.depart(u)
            live.discard(u)
        elif op < 0.85:
            p, d = rng.choice([0, 0, rng.randint(1, 900)]), rng.randint(0, 3)
            ours.charge(u, prefill=p, decode=d)
            ref.serve(u, prompt=p, output=d)
        else:
            ranks = {r: k for k, r in enumerate(rng.sample(range(12), 12))}
            queued = rng.sample(range(12), rng.randint(0, 12))
            slots = sorted(ranks[r] for r in queued)
            ours.redeal(ranks, queued)
            assert [r for s in slots for r in ranks if ranks[r] == s] == ref.order(queued)
        assert all(ours.get(i) == ref.counter(i) for i in range(12))
        assert ours.last_left == ref.l


@pytest.mark.parametrize("seed", range(12))
def test_paper_setting_matches_oracle_and_keeps_the_fairness_bound(seed):
    reqs, cap = _requests(seed)
    want, _ = vo.paper_server(reqs, cap, 1500)
    got, _ = vo.paper_server(reqs, cap, 1500, vtc_factory=_ProductVTC)
    assert got == want  # admissions, counters, service: step for step
    bound = vo.fairness_bound(1, 2, 256, cap)
    for _, counters, _, _ in got:
        if len(counters) > 1:
            assert max(counters.values()) - min(counters.values()) <= bound
    # service of two continuously backlogged clients differs by <= 2U
    for a in range(len(got)):
        for b in range(a + 1, min(len(got), a + 400), 37):
            both = set(got[a][1]) & set(got[b][1])
            if all(both <= set(got[k][1]) for k in range(a, b + 1)) and len(both) > 1:
                served = {u: got[b][1][u] - got[a][1][u] for u in both}
                assert max(served.values()) - min(served.values()) <= 2 * bound


def _vtc_run(doc):
    cfg, wl, _ = mconfig.build(doc)
    eng = Engine(cfg, generate(wl))
    gaps = []
    orig = eng._maybe_new_epoch

    def hook():
        orig()
        live = eng._live_ids()
        if len(live) > 1:
            cs = [eng.vtc.get(r) for r in live]
            gaps.append(max(cs) - min(cs))

    eng._maybe_new_epoch = hook
    return eng, json.loads(eng.run().to_json()), gaps


CONFIG3 = {"ablation": "full", "block": {"bytes_per_block": 2097152},
           "gpu_pool": {"total_blocks": 256},
           "workload": {"num_conversations": 30, "arrival_rate_per_s": 3.0},
           "trace": {"pattern": "vtc", "frequency": 0.04}}


def test_vtc_engine_run_conserves_tokens_and_is_deterministic():
    eng, rep, gaps = _vtc_run(CONFIG3)
    assert rep["total_tokens"] == rep["expected_tokens"]
    assert rep["swap_out_blocks"] > 0  # preemption happened under this pressure
    _, rep2, _ = _vtc_run(CONFIG3)
    assert rep2 == rep
    # every client was charged w_p per prompt token and w_q per output token
    # (plus lifts, which only raise counters)
    prompts = sum(t[0] for c in eng.conversations for t in c.turns)
    assert sum(eng.vtc.counters.values()) >= prompts + 2 * rep["total_tokens"]
    # VTC's bound holds among live clients with M = the GPU pool's tokens
    longest = max(t[0] for c in eng.conversations for t in c.turns)
    bound = vo.fairness_bound(1, 2, longest, 256 * 16)
    assert gaps and max(gaps) <= bound


def _random_vtc_doc(seed):
    r = random.Random(1000 + seed)
    blocks = r.choice([256, 384, 512])
    return {
        "ablation": r.choice(["baseline", "blockgroup", "blockgroup_reuse", "full"]),
        "gpu_pool": {"total_blocks": blocks,
                     "victim_policy": r.choice(["random", "lowest_priority"])},
        "cpu_pool": {"total_blocks": r.choice([1500, 16384])},
        "workload": {"num_conversations": r.randint(8, 40),
                     "arrival_rate_per_s": r.choice([1.0, 2.0, 4.0]),
                     "think_time_mean_s": r.choice([1.0, 2.0, 10.0]),
                     "max_context_tokens": blocks * 16},
        "trace": {"pattern": "vtc", "frequency": r.choice([0.0, 0.02, 0.04, 0.2]),
                  "vtc_wp": r.choice([1, 2]), "vtc_wq": r.choice([1, 2, 4])},
        "block": {"bytes_per_block": r.choice([131072, 2097152])},
        "seed": r.randint(0, 1000),
    }


@pytest.mark.parametrize("seed", range(int(os.environ.get("KVS_DIFF_SEEDS", "12"))))
def test_vtc_decisions_match_reference_engine_with_oracle_vtc(kvswitch, seed):
    from kvswitch import config as C
    from kvswitch import engine as ref_engine

    from test_differential_reference import _trace

    doc = _random_vtc_doc(seed)
    rdoc, wp, wq = vo.reference_doc(doc)
    s = C.build(rdoc)
    cfg, wl, _ = mconfig.build(doc)
    try:
        want = _trace(vo.vtc_reference_engine(ref_engine, wp, wq)(
            s.engine, kvswitch.generate(s.workload)))
    except Exception as exc:  # pool too small, deadlock: ours must fail the same way
        with pytest.raises(Exception) as ours:
            _trace(Engine(cfg, generate(wl)))
        assert type(ours.value).__name__ == type(exc).__name__
        assert str(ours.value).splitlines()[:1] == str(exc).splitlines()[:1]
        return
    got = _trace(Engine(cfg, generate(wl)))
    assert got[0] == want[0]
    assert got[1:] == want[1:]
