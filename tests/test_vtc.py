"""VTC (virtual token counter) priority pattern — the builder's addition for
BASELINE config 3; the reference has no oracle for it, so these
are property tests: least-served first, deterministic, tokens conserved."""

import json

from paper_2411_18424_b200 import config as mconfig
from paper_2411_18424_b200.engine import Engine
from paper_2411_18424_b200.scheduler import PriorityTrace, apply_priority_update
from paper_2411_18424_b200.workload import generate


def test_vtc_ranks_least_served_first_ties_by_id():
    trace = PriorityTrace(pattern="vtc", frequency=0.1)
    ranks = apply_priority_update(3, trace, live=[7, 2, 9, 4], running=[2, 9],
                                  served={7: 50, 2: 10, 9: 10, 4: 0})
    assert ranks == {4: 0, 2: 1, 9: 2, 7: 3}
    # RNG-free: the epoch number and the running set do not matter
    assert apply_priority_update(99, trace, [7, 2, 9, 4], [], {7: 50, 2: 10, 9: 10, 4: 0}) == ranks
    assert apply_priority_update(1, trace, [5, 1], [], None) == {1: 0, 5: 1}


def _run(pattern):
    cfg, wl, _ = mconfig.build({
        "ablation": "full", "block": {"bytes_per_block": 2097152},
        "gpu_pool": {"total_blocks": 256},
        "workload": {"num_conversations": 30, "arrival_rate_per_s": 3.0},
        "trace": {"pattern": pattern, "frequency": 0.04}})
    eng = Engine(cfg, generate(wl))
    rep = eng.run()
    return eng, json.loads(rep.to_json())


def test_vtc_engine_run_conserves_tokens_and_is_deterministic():
    eng, rep = _run("vtc")
    assert rep["total_tokens"] == rep["expected_tokens"]
    assert rep["swap_out_blocks"] > 0  # preemption happened under this pressure
    _, rep2 = _run("vtc")
    assert rep2 == rep
    # the engine fed VTC the tokens each request was served
    assert sum(eng.served_tokens.values()) == rep["total_tokens"]
