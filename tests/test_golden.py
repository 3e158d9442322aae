"""Control-plane parity against golden fixtures recorded from the reference
(oracle/gen_golden.py).  Runs anywhere — including the GPU box, where
/root/reference is absent.  Bar: bit-exact (integer / index work)."""

import json
from pathlib import Path

import pytest

from oracle import gen_golden as gg
from paper_2411_18424_b200 import alloc, cpu_store
from paper_2411_18424_b200 import config as mconfig
from paper_2411_18424_b200.alloc import PoolConfig
from paper_2411_18424_b200.engine import Engine, EngineConfig
from paper_2411_18424_b200.scheduler import (Candidate, PriorityTrace, SchedulerConfig,
                                             apply_priority_update, schedule)
from paper_2411_18424_b200.workload import Conversation, LengthDist, WorkloadConfig, generate

GOLD = Path(__file__).resolve().parent / "golden"


def load(name):
    return json.loads((GOLD / name).read_text())


@pytest.mark.parametrize("case", load("alloc.json")["cases"], ids=lambda c: str(c[0]))
def test_alloc_sequences_match_reference(case):
    args, want = case
    got = gg.alloc_sequence(alloc, *args)
    assert got["final_dump"] == want["final_dump"]
    assert got["trail_sha256"] == want["trail_sha256"]
    assert list(got["granularity"] or []) == list(want["granularity"] or [])


@pytest.mark.parametrize("case", load("cpu_store.json")["cases"], ids=lambda c: str(c[0]))
def test_cpu_store_sequences_match_reference(case):
    args, want = case
    assert gg.cpu_store_sequence(cpu_store, *args) == want


def test_priority_updates_match_reference():
    for pattern, seed, epoch, items in load("scheduler.json")["updates"]:
        live = list(range(0, 40, 3))
        trace = PriorityTrace(pattern=pattern, seed=seed, p_keep=0.8)
        got = apply_priority_update(epoch, trace, live, live[::2])
        assert sorted(got.items()) == [tuple(x) for x in items]


def test_schedules_match_reference():
    for cands, cap, cfg, want in load("scheduler.json")["schedules"]:
        cs = [Candidate(**c) for c in cands]
        a = schedule(cs, cap, SchedulerConfig(**cfg))
        assert [a.admit, a.swap_in, a.swap_out] == want


def test_workload_generation_matches_reference():
    for case in load("workload.json"):
        kwargs = {}
        if case["long"]:
            kwargs = dict(input_tokens=LengthDist(6000.0, 0.9, 16384),
                          output_tokens=LengthDist(112.0, 0.7, 512))
        convs = generate(WorkloadConfig(num_conversations=case["n"], seed=case["seed"],
                                        max_context_tokens=case["ctx"], **kwargs))
        rows = [[c.id, [list(t) for t in c.turns], c.arrival, c.think_time] for c in convs]
        assert gg.h(rows) == case["sha256"]


def _engine_for(name, doc):
    if doc is None:
        cfg = EngineConfig(gpu_pool=PoolConfig(total_blocks=48, initial_group_blocks=20),
                           trace=PriorityTrace(pattern="random", frequency=0.2, seed=1),
                           ablation="full")
        convs = [Conversation(0, [(320, 320)], 0, 0), Conversation(1, [(320, 320)], 1000, 0)]
        return Engine(cfg, convs)
    cfg, wl, _ = mconfig.build(doc)
    return Engine(cfg, generate(wl))


@pytest.mark.parametrize("name", sorted(load("engine.json")))
def test_engine_matches_reference(name, monkeypatch):
    want = load("engine.json")[name]
    if want.get("deadlock_iterations"):  # config 5: engine.py:48 patched in both engines
        from paper_2411_18424_b200 import engine as engine_mod
        monkeypatch.setattr(engine_mod, "DEADLOCK_ITERATIONS", want["deadlock_iterations"])
    eng = _engine_for(name, want["doc"])
    plans = []
    orig = eng.manager.dispatch

    def spy(clock, iteration, plan, not_before=0):
        plans.append([iteration, plan.request, plan.direction, plan.moved_blocks,
                      plan.reused_blocks, [[o.blocks, o.gpu_start, o.cpu_start]
                                           for o in plan.ops], not_before])
        return orig(clock, iteration, plan, not_before)

    eng.manager.dispatch = spy
    report = json.loads(eng.run().to_json())
    assert report == want["report"]
    events = [[e.iteration, e.request, e.direction, e.ops, e.blocks, e.dispatch_done,
               e.exec_done] for e in eng.manager.events_log]
    assert gg.h(events) == want["events_sha256"]
    assert plans[:20] == want["first_plans"]
    assert gg.h(plans) == want["plans_sha256"]
    assert gg.h(eng.pool.dump()) == want["gpu_dump_sha256"]
    assert gg.h(eng.store.dump()) == want["cpu_dump_sha256"]
