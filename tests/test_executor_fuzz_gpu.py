"""Randomized hazard test of the StreamExecutor: compute writes, swap-outs and
swap-ins on overlapping GPU and host extents, issued without host syncs,
must leave exactly what a sequential (program-order) numpy model leaves.
Exercises the cross-stream waits (compute -> both directions, WAR/RAW/WAW
between directions, op- and plane-granular compute barriers)."""

import os

import numpy as np
import pytest

from oracle import bytes_oracle as orc

pytestmark = pytest.mark.gpu


def _extent_ops(rng, G, C, max_ops=3, max_len=6):
    """1..max_ops TransferOps at random positions; ops overlapping an earlier
    op of the same plan (GPU or host side) are dropped."""
    from paper_2411_18424_b200.cpu_store import TransferOp

    kept = []
    for _ in range(int(rng.integers(1, max_ops + 1))):
        L = int(rng.integers(1, max_len + 1))
        op = TransferOp(L, int(rng.integers(0, G - L + 1)), int(rng.integers(0, C - L + 1)))
        if all(op.gpu_start + L <= k.gpu_start or k.gpu_start + k.blocks <= op.gpu_start
               for k in kept) and \
           all(op.cpu_start + L <= k.cpu_start or k.cpu_start + k.blocks <= op.cpu_start
               for k in kept):
            kept.append(op)
    return kept


SEEDS = int(os.environ.get("KVS_FUZZ_SEEDS", "1"))  # more for a soak run


@pytest.mark.parametrize("seed", range(SEEDS))
@pytest.mark.parametrize("mode", ["ops", "layered", "bulk", "bulk_ops", "bulk_layered",
                                  "partition", "staged", "mix"])
def test_random_interleavings_match_program_order(cuda_ok, mode, seed):
    torch = cuda_ok
    from paper_2411_18424_b200.dataplane import HostKVPool, PagedKVCache, SwapDataPlane
    from paper_2411_18424_b200.geometry import KVGeometry
    from paper_2411_18424_b200.swap import StreamExecutor

    geo = KVGeometry("fuzz", num_layers=3, num_kv_heads=1, head_dim=512)  # 32 KiB chunks
    G = C = 48
    cache = PagedKVCache(geo, G, device="cuda:0")
    host = HostKVPool(C, geo.block_bytes)
    dp = SwapDataPlane(cache, host)
    policy = {"bulk": "throughput", "bulk_ops": "latency_bulk",
              "bulk_layered": "latency_bulk", "staged": "throughput_staged",
              "mix": "throughput_mix"}.get(mode, "latency")
    if mode in ("staged", "mix"):
        dp.set_staging(2 * geo.block_bytes, 2)  # tiny ring: plans span slots, slots recycle
    ex = StreamExecutor(dp, duplex_policy=policy, layered_swap_in=mode.endswith("layered"),
                        sm_partition=8 if mode == "partition" else 0)
    assert ex.op_granular == (mode not in ("bulk", "staged", "mix"))
    rng = np.random.default_rng([{"ops": 1, "layered": 2, "bulk": 3, "partition": 4,
                                  "bulk_ops": 5, "bulk_layered": 6, "staged": 7,
                                  "mix": 8}[mode], seed])
    last_in = None
    gpu = np.zeros((geo.num_planes, G, geo.plane_chunk_bytes), np.uint8)
    hostm = np.zeros((C, geo.block_bytes), np.uint8)
    cache.planes.zero_()
    host.array[:] = 0
    torch.cuda.synchronize()
    for step in range(400):
        a = rng.random()
        if a < 0.35:  # compute writes one value into a GPU extent
            L = int(rng.integers(1, 5))
            s = int(rng.integers(0, G - L + 1))
            val = int(rng.integers(1, 255))
            ex.compute_barrier([(s, L)])
            with torch.cuda.stream(ex.compute):
                if rng.random() < 0.5:
                    torch.cuda._sleep(300_000)  # compute lags: later swaps must still wait
                cache.planes[:, s:s + L].fill_(val)
            gpu[:, s:s + L] = val
        elif a < 0.7:
            ops = _extent_ops(rng, G, C)
            ex.submit("out", ops)
            orc.apply_plan("out", gpu, hostm, [(o.blocks, o.gpu_start, o.cpu_start) for o in ops])
        elif a < 0.9 or last_in is None or not mode.endswith("layered"):
            ops = _extent_ops(rng, G, C)
            last_in = (ex.submit("in", ops), ops)
            orc.apply_plan("in", gpu, hostm, [(o.blocks, o.gpu_start, o.cpu_start) for o in ops])
        else:
            # layered join: compute writes plane l of the latest swap-in's blocks as
            # soon as plane l has landed (kvs_swap_signaled plane flags)
            rec, ops = last_in
            # as the engine does: other transfers on these blocks per op, the
            # joining swap-in itself per plane
            ex.compute_barrier([(o.gpu_start, o.blocks) for o in ops], skip=(rec,))
            with torch.cuda.stream(ex.compute):
                torch.cuda._sleep(100_000)
            for plane in range(geo.num_planes):
                ex.wait_plane(ex.compute, rec, plane)
                val = int(rng.integers(1, 255))
                with torch.cuda.stream(ex.compute):
                    for o in ops:
                        cache.planes[plane, o.gpu_start:o.gpu_start + o.blocks].fill_(val)
                for o in ops:
                    gpu[plane, o.gpu_start:o.gpu_start + o.blocks] = val
            last_in = None
        if step % 97 == 96:
            ex.synchronize()
            np.testing.assert_array_equal(cache.planes.cpu().numpy(), gpu)
            np.testing.assert_array_equal(host.array, hostm)
    ex.synchronize()
    np.testing.assert_array_equal(cache.planes.cpu().numpy(), gpu)
    np.testing.assert_array_equal(host.array, hostm)
    assert dp.launches > 100  # swap kernels, or the staged path's gather / scatter kernels
    host.close()
