"""Differential parity against the live reference (this container only; the
GPU box uses the committed goldens): random engine configurations —
ablation, pool sizes, first-group size, victim policy, host pool, scheduler
caps, preemption mode, priority pattern, workload shape — run through the
reference's Engine and through ours must give the same MetricsReport, the
same SwapEvent log and the same dispatched plan stream (every TransferOp)."""

import json
import os
import random

import pytest

from oracle import gen_golden as gg
from paper_2411_18424_b200 import config as mconfig
from paper_2411_18424_b200.engine import Engine
from paper_2411_18424_b200.workload import generate


def _random_doc(seed):
    r = random.Random(seed)
    doc = {
        "ablation": r.choice(["baseline", "blockgroup", "blockgroup_reuse", "full"]),
        "gpu_pool": {"total_blocks": r.choice([160, 256, 384, 512, 1024]),
                     "initial_group_blocks": r.choice([8, 20, 60, 100]),
                     "victim_policy": r.choice(["random", "lowest_priority"])},
        "cpu_pool": {"total_blocks": r.choice([1500, 4000, 16384])},
        "workload": {"num_conversations": r.randint(8, 36),
                     "arrival_rate_per_s": r.choice([0.5, 1.0, 2.0, 4.0]),
                     "think_time_mean_s": r.choice([1.0, 5.0, 10.0])},
        "trace": {"pattern": r.choice(["markov", "random"]),
                  "frequency": r.choice([0.0, 0.02, 0.04, 0.2])},
        "block": {"bytes_per_block": r.choice([131072, 655360, 2097152])},
        "seed": r.randint(0, 1000),
    }
    if r.random() < 0.3:
        doc["scheduler"] = {"max_running": r.choice([4, 8, 16])}
    if r.random() < 0.2:
        doc.setdefault("scheduler", {})["preemption_mode"] = "recompute"
    return doc


def _trace(eng):
    plans = []
    orig = eng.manager.dispatch

    def spy(clock, iteration, plan, not_before=0):
        plans.append([iteration, plan.request, plan.direction, plan.moved_blocks,
                      plan.reused_blocks, [[o.blocks, o.gpu_start, o.cpu_start]
                                           for o in plan.ops], not_before])
        return orig(clock, iteration, plan, not_before)

    eng.manager.dispatch = spy
    report = json.loads(eng.run().to_json())
    events = [[e.iteration, e.request, e.direction, e.ops, e.blocks, e.dispatch_done,
               e.exec_done] for e in eng.manager.events_log]
    return report, gg.h(events), gg.h(plans), gg.h(eng.pool.dump()), gg.h(eng.store.dump())


@pytest.mark.parametrize("seed", range(int(os.environ.get("KVS_DIFF_SEEDS", "16"))))
def test_random_configurations_match_the_reference(kvswitch, seed):
    from kvswitch import config as C
    from kvswitch.engine import Engine as RefEngine

    doc = _random_doc(seed)
    try:
        s = C.build(doc)
    except ValueError as exc:  # the reference rejects it: so must we
        with pytest.raises(ValueError):
            mconfig.build(doc)
        pytest.skip(f"reference rejects the document: {exc}")
    try:
        want = _trace(RefEngine(s.engine, kvswitch.generate(s.workload)))
    except Exception as exc:  # e.g. DeadlockError, pool too small
        cfg, wl, _ = mconfig.build(doc)
        with pytest.raises(type(exc)):
            Engine(cfg, generate(wl)).run()
        return
    cfg, wl, _ = mconfig.build(doc)
    got = _trace(Engine(cfg, generate(wl)))
    assert got[0] == want[0]  # MetricsReport
    assert got[1:] == want[1:]  # event log, plan stream, final pool dumps
