"""N>1 path on CPU: world_size-2 gloo processes, each a TP rank of a sharded
KV cache, run the replicated control plane and agree on the plan stream;
timing aggregates as max over ranks (bench.py rule)."""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2411_18424_b200 import config as mconfig
        from paper_2411_18424_b200 import multirank
        from paper_2411_18424_b200.engine import Engine
        from paper_2411_18424_b200.geometry import QWEN25_32B
        from paper_2411_18424_b200.workload import generate

        geo = multirank.shard(QWEN25_32B, world)
        lo, hi = geo.head_slice(rank)
        cfg, wl, _ = mconfig.build({
            "ablation": "full", "block": {"bytes_per_block": geo.block_bytes},
            "gpu_pool": {"total_blocks": 256},
            "workload": {"num_conversations": 20, "arrival_rate_per_s": 3.0},
            "trace": {"pattern": "random", "frequency": 0.04}})
        eng = Engine(cfg, generate(wl))
        dig = multirank.PlanDigest().attach(eng.manager)
        rep = eng.run()
        same = multirank.agree(dig.hexdigest())
        t = multirank.max_over_ranks(float(rank + 1))
        total_bytes = multirank.sum_over_ranks(float(geo.block_bytes))
        q.put((rank, same, t, total_bytes, (lo, hi), dig.plans, rep.swap_out_blocks))
    finally:
        dist.destroy_process_group()


def test_two_rank_tp_shards_agree_on_plans():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got.sort()
    from paper_2411_18424_b200.geometry import QWEN25_32B

    for rank, same, t, total, heads, plans, blocks in got:
        assert same, "ranks dispatched different plan streams"
        assert t == 2.0  # max over ranks
        assert total == QWEN25_32B.block_bytes  # shards sum to the model's block
        assert plans > 0
    assert [g[4] for g in got] == [(0, 4), (4, 8)]  # head shards partition 8 KV heads
    assert got[0][6] == got[1][6]


def _agree_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2411_18424_b200.live import RankAgreement

        ag = RankAgreement()
        # rank 1's clock runs ahead; a swap counts as landed only once it landed everywhere
        flags = [[True, False, True, True], [True, True, False, True]][rank]
        clock, landed = ag.landed(1000 + 500 * rank, flags)
        end = ag.clock(7 - rank)
        empty = ag.landed(3, [])
        q.put((rank, clock, landed, end, empty, ag.calls))
    finally:
        dist.destroy_process_group()


def test_rank_agreement_max_clock_and_all_landed():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_agree_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, clock, landed, end, empty, calls in got:
        assert clock == 1500
        assert landed == [True, False, False, True]
        assert end == 7
        assert empty == (3, [])
        assert calls == 3
