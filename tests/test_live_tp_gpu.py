"""Live mode across a TP group: two ranks (two processes sharing cuda:0, gloo
for the control-plane agreement) each swap their own KV-head shard, agree on
clock and landed swaps every iteration, and must therefore take identical
decisions: same plan stream, same TTFT/TBT samples.  Bytes are verified on
every swap-in of every rank."""

import os
import socket

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q, layered=False):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2411_18424_b200 import multirank
        from paper_2411_18424_b200.alloc import PoolConfig
        from paper_2411_18424_b200.engine import EngineConfig
        from paper_2411_18424_b200.geometry import LLAMA3_8B
        from paper_2411_18424_b200.live import (DecodeEmulator, LiveEngine, RankAgreement,
                                                b200_transfer_params)
        from paper_2411_18424_b200.runtime import Runtime
        from paper_2411_18424_b200.scheduler import PriorityTrace
        from paper_2411_18424_b200.workload import WorkloadConfig, generate

        geo = LLAMA3_8B.with_tp(world)
        convs = generate(WorkloadConfig(num_conversations=10, seed=5, max_context_tokens=2048,
                                        arrival_rate_per_s=20.0, think_time_mean_s=0.05))
        cfg = EngineConfig(gpu_pool=PoolConfig(total_blocks=128, initial_group_blocks=40),
                           trace=PriorityTrace(pattern="random", frequency=0.04, seed=2),
                           ablation="full", cpu_pool_blocks=2048,
                           transfer=b200_transfer_params())
        rt = Runtime(geo, 128, 2048, device="cuda:0", verify=True, timing=True,
                     layered_swap_in=layered)
        dec = DecodeEmulator("cuda:0", weight_bytes=1 << 30)
        eng = LiveEngine(cfg, convs, rt, dec, agreement=RankAgreement(), layered=layered)
        dig = multirank.PlanDigest().attach(eng.manager)
        rep = eng.run()
        q.put((rank, dig.hexdigest(), dig.plans, list(eng.ttft_samples),
               list(eng.tbt_samples), rep.total_tokens, rep.expected_tokens,
               rt.verified, rt.stats()["bytes_out"], eng.agreement.calls))
        rt.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,layered", [(2, False), (2, True), (4, True)])
def test_two_tp_ranks_decide_in_lockstep(cuda_ok, world, layered):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, layered))
             for r in range(world)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    r0 = got[0]
    _, d0, n0, ttft0, tbt0, tok0, exp0, ver0, out0, calls0 = r0
    assert n0 > 0 and tok0 == exp0
    for _, d, n, ttft, tbt, tok, _, ver, out, calls in got[1:]:
        assert d == d0 and n == n0  # identical plan streams
        assert ttft == ttft0 and tbt == tbt0  # identical agreed timestamps
        assert tok == tok0 and calls == calls0
        assert out == out0 > 0  # equal shard sizes -> equal bytes per rank
    assert all(g[7] > 0 for g in got)  # every rank's swap-ins verified byte-exact
