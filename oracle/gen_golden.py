"""ORACLE — golden-fixture generator (test infrastructure; run in the build
container where the reference is mounted read-only at /root/reference).

Imports the UNMODIFIED reference package (kvswitch, pkg/src) and records its
outputs on seeded inputs into tests/golden/*.json, so parity can be checked
on the GPU box where /root/reference does not exist:

  * engine.json   — full MetricsReport + digests of the SwapEvent log and of
                    the dispatched SwapPlan stream (every TransferOp) for a
                    set of engine configurations (engine.py:351-554,
                    swap.py:181-232, cpu_store.py:209-337);
  * alloc.json    — BlockGroupPool.dump() digests along seeded op sequences
                    (alloc.py:218-532), both victim policies;
  * cpu_store.json— plan digests along seeded CpuStore op sequences;
  * scheduler.json— apply_priority_update / schedule outputs (scheduler.py);
  * workload.json — generate() digests (workload.py:97-124).

Usage:  python oracle/gen_golden.py            (writes tests/golden/)
"""

from __future__ import annotations

import hashlib
import json
import random
import sys
from pathlib import Path

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parents[1] / "tests" / "golden"


def h(obj) -> str:
    return hashlib.sha256(json.dumps(obj, sort_keys=True).encode()).hexdigest()


# Engine configurations (config.py document overrides). Shared with the tests.
ENGINE_CASES = {
    "duel_full": None,  # test_engine.py small_cfg + duel_conversations, built below
    "default_baseline": {"ablation": "baseline", "workload": {"num_conversations": 60}},
    "default_blockgroup": {"ablation": "blockgroup", "workload": {"num_conversations": 60}},
    "default_reuse": {"ablation": "blockgroup_reuse", "workload": {"num_conversations": 60}},
    "default_full": {"ablation": "full", "workload": {"num_conversations": 60}},
    "pressure_random": {"ablation": "full", "gpu_pool": {"total_blocks": 256},
                        "workload": {"arrival_rate_per_s": 3.0, "num_conversations": 60},
                        "trace": {"pattern": "random", "frequency": 0.04}},
    "cpu_tight_lowprio": {"ablation": "full",
                          "gpu_pool": {"total_blocks": 300, "victim_policy": "lowest_priority"},
                          "cpu_pool": {"total_blocks": 2000},
                          "workload": {"arrival_rate_per_s": 2.0, "num_conversations": 60}},
    "caps_reuse": {"ablation": "blockgroup_reuse", "gpu_pool": {"total_blocks": 256},
                   "scheduler": {"max_running": 8, "max_prefill_tokens": 2048},
                   "workload": {"num_conversations": 60}},
    "recompute": {"ablation": "full", "gpu_pool": {"total_blocks": 256},
                  "scheduler": {"preemption_mode": "recompute"},
                  "workload": {"num_conversations": 40}},
    "llama8b_2mib": {"ablation": "full", "block": {"bytes_per_block": 2097152},
                     "gpu_pool": {"total_blocks": 512},
                     "transfer": {"bandwidth_bytes_per_us": 63000},
                     "workload": {"arrival_rate_per_s": 2.0, "num_conversations": 60},
                     "trace": {"pattern": "markov", "frequency": 0.04}},
    # BASELINE config 3: VTC priorities (reference engine + oracle/vtc_oracle.py)
    "vtc_config3_bench": {"ablation": "full", "block": {"bytes_per_block": 2097152},
                          "gpu_pool": {"total_blocks": 512}, "cpu_pool": {"total_blocks": 4096},
                          "workload": {"num_conversations": 64, "arrival_rate_per_s": 4.0,
                                       "think_time_mean_s": 2.0},
                          "trace": {"pattern": "vtc", "frequency": 0.04}},
    "vtc_config3_default": {"ablation": "full", "block": {"bytes_per_block": 2097152},
                            "gpu_pool": {"total_blocks": 512},
                            "cpu_pool": {"total_blocks": 8192},
                            "workload": {"num_conversations": 200, "arrival_rate_per_s": 2.0},
                            "trace": {"pattern": "vtc", "frequency": 0.04}},
    "vtc_config3_baseline": {"ablation": "baseline", "block": {"bytes_per_block": 2097152},
                             "gpu_pool": {"total_blocks": 512},
                             "cpu_pool": {"total_blocks": 4096},
                             "workload": {"num_conversations": 64, "arrival_rate_per_s": 4.0,
                                          "think_time_mean_s": 2.0},
                             "trace": {"pattern": "vtc", "frequency": 0.04}},
    "vtc_pressure_lowprio": {"ablation": "full",
                             "gpu_pool": {"total_blocks": 256,
                                          "victim_policy": "lowest_priority"},
                             "cpu_pool": {"total_blocks": 1500},
                             "workload": {"arrival_rate_per_s": 3.0, "num_conversations": 60},
                             "trace": {"pattern": "vtc", "frequency": 0.2,
                                       "vtc_wp": 1, "vtc_wq": 4}},
}
# BASELINE config 4: Qwen-2.5-32B KV, per-rank shard bytes at TP 2/4/8
# (64 layers x 8 KV heads x d 128 x 16 tok x 2 (K,V) x fp16 / TP), multi-turn
# reuse, random priorities f=0.04.
for _tp in (2, 4, 8):
    ENGINE_CASES[f"c4_qwen32b_tp{_tp}"] = {
        "ablation": "full", "block": {"bytes_per_block": 4194304 // _tp},
        "gpu_pool": {"total_blocks": 1024}, "cpu_pool": {"total_blocks": 8192},
        "workload": {"num_conversations": 60, "arrival_rate_per_s": 2.0},
        "trace": {"pattern": "random", "frequency": 0.04}}
# BASELINE config 5: LLaMA-3-70B TP8 rank shard (655360 B per block), 32K
# context, high preemption.  The reference's deadlock detector fires on
# legitimately long swaps here (engine.py:48, :536-538): both engines run it
# with DEADLOCK_ITERATIONS = 1000.
ENGINE_CASES["c5_llama70b_tp8"] = {
    "ablation": "full", "block": {"bytes_per_block": 655360},
    "gpu_pool": {"total_blocks": 8192, "initial_group_blocks": 60},
    "cpu_pool": {"total_blocks": 65536},
    "workload": {"num_conversations": 64, "arrival_rate_per_s": 1.0,
                 "input_tokens": {"median": 6000.0, "sigma": 0.9, "max": 16384},
                 "max_context_tokens": 32768},
    "trace": {"pattern": "random", "frequency": 0.04}}
DEADLOCK_ITERATIONS = {"c5_llama70b_tp8": 1000}


def engine_goldens(kv):
    from kvswitch import config as C
    from kvswitch import engine as ref_engine
    from kvswitch.alloc import PoolConfig
    from kvswitch.engine import Engine, EngineConfig
    from kvswitch.scheduler import PriorityTrace
    from kvswitch.workload import Conversation

    from oracle import vtc_oracle

    out = {}
    for name, doc in ENGINE_CASES.items():
        make = Engine
        if doc is not None and doc.get("trace", {}).get("pattern") == "vtc":
            ref_doc, wp, wq = vtc_oracle.reference_doc(doc)
            make = vtc_oracle.vtc_reference_engine(ref_engine, wp, wq)
        else:
            ref_doc = doc
        if doc is None:
            cfg = EngineConfig(gpu_pool=PoolConfig(total_blocks=48, initial_group_blocks=20),
                               trace=PriorityTrace(pattern="random", frequency=0.2, seed=1),
                               ablation="full")
            convs = [Conversation(0, [(320, 320)], 0, 0), Conversation(1, [(320, 320)], 1000, 0)]
            settings_doc = {"special": "duel"}
        else:
            s = C.build(ref_doc)
            cfg, convs, settings_doc = s.engine, kv.generate(s.workload), s.doc
        eng = make(cfg, convs)
        plans = []
        orig = eng.manager.dispatch

        def spy(clock, iteration, plan, not_before=0, _orig=orig, _plans=plans):
            _plans.append([iteration, plan.request, plan.direction, plan.moved_blocks,
                           plan.reused_blocks, [[o.blocks, o.gpu_start, o.cpu_start]
                                                for o in plan.ops], not_before])
            return _orig(clock, iteration, plan, not_before)

        eng.manager.dispatch = spy
        saved = ref_engine.DEADLOCK_ITERATIONS
        ref_engine.DEADLOCK_ITERATIONS = DEADLOCK_ITERATIONS.get(name, saved)
        try:
            report = eng.run()
        finally:
            ref_engine.DEADLOCK_ITERATIONS = saved
        events = [[e.iteration, e.request, e.direction, e.ops, e.blocks, e.dispatch_done,
                   e.exec_done] for e in eng.manager.events_log]
        out[name] = {"doc": doc, "deadlock_iterations": DEADLOCK_ITERATIONS.get(name),
                     "report": json.loads(report.to_json()),
                     "events_sha256": h(events), "plans_sha256": h(plans),
                     "n_events": len(events), "first_plans": plans[:20],
                     "gpu_dump_sha256": h(eng.pool.dump()),
                     "cpu_dump_sha256": h(eng.store.dump())}
        print(f"engine {name}: {report.iterations} iterations, {len(events)} swaps", flush=True)
    return out


def alloc_sequence(mod, seed: int, total: int, initial: int, policy: str, steps: int):
    """Seeded mixed sequence: allocate / fill / free_group / free_request /
    reclaim / allocate_at / shrink; dump digest every 200 steps."""
    PoolConfig, Pool = mod.PoolConfig, mod.BlockGroupPool
    pool = Pool(PoolConfig(total_blocks=total, initial_group_blocks=initial, rng_seed=seed,
                           victim_policy=policy))
    ranks = {}
    pool.rank_of = lambda r: ranks.get(r, 1 << 30)
    rng = random.Random(seed * 7919 + total)
    live, nxt, trail = [], 0, []
    for step in range(steps):
        roll = rng.random()
        try:
            if roll < 0.4 or not live:
                req = nxt
                nxt += 1
                ranks[req] = rng.randint(0, 50)
                want = rng.randint(1, max(1, total // 12))
                exp = want + rng.randint(0, 80) if rng.random() < 0.7 else None
                res = pool.allocate(req, want, expected_total=exp, reclaim=rng.random() < 0.8)
                live.append(req)
                pool.set_request_fill(req, rng.randint(0, res.total_blocks))
                trail.append(["a", [(g.start, g.length, g.id) for g in res.groups],
                              res.reclaimed_from])
            elif roll < 0.55:
                req = rng.choice(live)
                more = rng.randint(1, 20)
                res = pool.allocate(req, more, expected_total=more + rng.randint(0, 30))
                pool.set_request_fill(req, rng.randint(0, pool.owned_blocks(req)))
                trail.append(["g", [(g.start, g.length, g.id) for g in res.groups]])
            elif roll < 0.75:
                req = rng.choice(live)
                trail.append(["f", pool.free_request(req)])
                live.remove(req)
            elif roll < 0.85:
                req = rng.choice(live)
                groups = pool.owned_groups(req)
                g = groups[rng.randrange(len(groups))]
                if rng.random() < 0.5 and g.length > 1:
                    pool.shrink_group(g.id, rng.randint(max(1, g.filled), g.length))
                    trail.append(["s", g.id])
                else:
                    pool.free_group(g.id)
                    trail.append(["fg", g.id])
                    if not pool.owned_groups(req):
                        live.remove(req)
            elif roll < 0.93:
                req = nxt
                nxt += 1
                owner, piece = pool.reclaim_from_victim(rng.randint(1, 12), for_request=req)
                live.append(req)
                trail.append(["r", owner, piece.start, piece.length, piece.id])
            else:
                req = nxt
                nxt += 1
                start = rng.randrange(total)
                g = pool.allocate_at(req, start, rng.randint(1, 16))
                if g is not None:
                    live.append(req)
                trail.append(["at", None if g is None else (g.start, g.length, g.id)])
        except Exception as exc:  # OOM / NoVictim are part of the contract
            trail.append(["x", type(exc).__name__])
        if step % 200 == 0:
            pool.validate()
            trail.append(["d", h(pool.dump())])
    return {"final_dump": pool.dump(), "trail_sha256": h(trail), "steps": steps,
            "granularity": pool.granularity_stats()}


ALLOC_CASES = [(1, 2048, 60, "random", 4000), (2, 512, 16, "random", 4000),
               (3, 1024, 40, "lowest_priority", 4000), (4, 300, 60, "random", 3000),
               (5, 64, 8, "lowest_priority", 3000)]


def cpu_store_sequence(mod, seed: int, total: int, reuse: bool, steps: int):
    Store = mod.CpuStore
    store = Store(total_blocks=total, reuse_enabled=reuse)
    rng = random.Random(seed)
    foot = {}
    trail = []
    for step in range(steps):
        req = rng.randrange(12)
        store.set_rank(req, rng.randint(0, 9))
        roll = rng.random()
        try:
            if roll < 0.5:
                fp = foot.get(req, 0) + rng.randint(0, 40)
                foot[req] = fp
                if fp == 0:
                    continue
                # GPU table: fp blocks in 1-4 runs at arbitrary positions
                cuts = sorted(rng.sample(range(1, fp), min(fp - 1, rng.randint(0, 3))))
                sizes = [b - a for a, b in zip([0] + cuts, cuts + [fp])]
                ext, pos = [], rng.randrange(10000)
                for s in sizes:
                    ext.append((pos, s))
                    pos += s + rng.randint(1, 50)
                plan = store.plan_swap_out(req, fp, ext)
                trail.append(["o", req, plan.moved_blocks, plan.reused_blocks,
                              [(o.blocks, o.gpu_start, o.cpu_start) for o in plan.ops]])
                if rng.random() < 0.6:
                    trail.append(["p", store.preallocate_increment(req, rng.randint(0, 64))])
            elif roll < 0.8:
                fp = foot.get(req, 0)
                if fp == 0:
                    continue
                ext = [(rng.randrange(5000), fp)]
                try:
                    plan = store.plan_swap_in(req, ext)
                    trail.append(["i", req, [(o.blocks, o.gpu_start, o.cpu_start)
                                             for o in plan.ops]])
                except mod.ContaminatedCopyError:
                    plan, pre = store.plan_swap_in_prefix(req, ext)
                    foot[req] = pre
                    trail.append(["ip", req, pre, [(o.blocks, o.gpu_start, o.cpu_start)
                                                   for o in plan.ops]])
            elif roll < 0.9:
                trail.append(["e", store.evict_for(rng.randint(0, 9), rng.randint(0, 30))])
            else:
                store.release(req)
                foot.pop(req, None)
                trail.append(["rel", req])
        except Exception as exc:
            trail.append(["x", type(exc).__name__])
        if step % 100 == 0:
            store.pool.validate()
            trail.append(["d", h(store.dump())])
    return {"trail_sha256": h(trail), "final_dump_sha256": h(store.dump()),
            "peak": store.peak_used_blocks}


CPU_CASES = [(11, 400, True, 3000), (12, 150, True, 3000), (13, 400, False, 2000),
             (14, 2000, True, 3000)]


def scheduler_goldens():
    from kvswitch.scheduler import Candidate, PriorityTrace, SchedulerConfig, \
        apply_priority_update, schedule
    out = {"updates": [], "schedules": []}
    for pattern in ("random", "markov"):
        for seed in (0, 1, 42):
            for epoch in (1, 2, 7):
                live = list(range(0, 40, 3))
                running = live[::2]
                trace = PriorityTrace(pattern=pattern, seed=seed, p_keep=0.8)
                r = apply_priority_update(epoch, trace, live, running)
                out["updates"].append([pattern, seed, epoch, sorted(r.items())])
    rng = random.Random(3)
    for _ in range(200):
        n = rng.randint(1, 12)
        cands = [Candidate(i, rng.randint(0, 20), rng.choice(
            ["running", "swapped", "waiting", "ongoing_swap_in"]), rng.randint(1, 60),
            rng.randint(0, 500)) for i in range(n)]
        cfg = SchedulerConfig(max_running=rng.choice([None, 3, 6]),
                              max_prefill_tokens=rng.choice([None, 300, 800]))
        cap = rng.randint(20, 200)
        a = schedule(cands, cap, cfg)
        out["schedules"].append([[c.__dict__ for c in cands], cap, cfg.__dict__,
                                 [a.admit, a.swap_in, a.swap_out]])
    return out


def workload_goldens(kv):
    from kvswitch.workload import LengthDist, WorkloadConfig, generate
    out = []
    for seed, n, ctx in ((0, 200, None), (5, 12, 2048), (42, 200, 3072), (9, 64, 32768)):
        kwargs = {}
        if ctx == 32768:
            kwargs = dict(input_tokens=LengthDist(6000.0, 0.9, 16384),
                          output_tokens=LengthDist(112.0, 0.7, 512))
        convs = generate(WorkloadConfig(num_conversations=n, seed=seed, max_context_tokens=ctx,
                                        **kwargs))
        rows = [[c.id, c.turns, c.arrival, c.think_time] for c in convs]
        out.append({"seed": seed, "n": n, "ctx": ctx, "long": ctx == 32768,
                    "sha256": h(rows), "head": rows[:3]})
    return out


def main():
    sys.path.insert(0, str(REF))
    sys.path.insert(0, str(OUT.parents[1]))
    import kvswitch as kv
    from kvswitch import alloc, cpu_store

    OUT.mkdir(parents=True, exist_ok=True)
    (OUT / "scheduler.json").write_text(json.dumps(scheduler_goldens()))
    (OUT / "workload.json").write_text(json.dumps(workload_goldens(kv), indent=1))
    (OUT / "alloc.json").write_text(json.dumps(
        {"cases": [[list(c), alloc_sequence(alloc, *c)] for c in ALLOC_CASES]}, indent=1))
    (OUT / "cpu_store.json").write_text(json.dumps(
        {"cases": [[list(c), cpu_store_sequence(cpu_store, *c)] for c in CPU_CASES]}, indent=1))
    (OUT / "engine.json").write_text(json.dumps(engine_goldens(kv), indent=1))
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()
