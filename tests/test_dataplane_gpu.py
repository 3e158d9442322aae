"""GPU parity of the swap kernels (K1 swap-out gather, K2 swap-in scatter)
against the oracle's TransferOp restatement (oracle/bytes_oracle.py), all
through the C ABI (libkvswap.so via paper_2411_18424_b200.dataplane).

Bar: bit-exact.  Small shapes are compared byte-for-byte with the numpy
oracle; BASELINE-size shapes use the round-trip property
(out -> poison HBM -> in to a different table == original).
"""

import numpy as np
import pytest

from oracle import bytes_oracle as orc

from conftest import under_sanitizer  # noqa: E402

pytestmark = pytest.mark.gpu


def _mk(torch, geometry, gpu_blocks, cpu_blocks, ctas=None, path="lsu", piece=0, stages=0):
    from paper_2411_18424_b200.dataplane import HostKVPool, PagedKVCache, SwapDataPlane

    cache = PagedKVCache(geometry, gpu_blocks, device="cuda:0")
    host = HostKVPool(cpu_blocks, geometry.block_bytes)
    plane = SwapDataPlane(cache, host, ctas=ctas)
    for d in ("out", "in"):
        plane.set_path(d, path, piece, stages)
    return cache, host, plane


PATHS = [("lsu", 0, 0), ("bulk", 0, 0), ("bulk", 4096, 2), ("bulk", 32768, 6)]


def _small_geometry(chunk_words=1028, planes=3):
    from paper_2411_18424_b200.geometry import KVGeometry

    # chunk = 2 (K,V) * 1 token * 1 head * d * 2 B = 4 * chunk_words bytes;
    # 1028 words -> 4112 B is not a multiple of the 4 KiB piece, which
    # exercises the ragged tail path.
    return KVGeometry("tiny", num_layers=planes, num_kv_heads=1, head_dim=chunk_words,
                      block_tokens=1)


@pytest.mark.parametrize("path", PATHS, ids=lambda p: f"{p[0]}-{p[1]}-{p[2]}")
@pytest.mark.parametrize("chunk_words,planes", [(1028, 3), (1024, 2), (4, 1), (16400, 5)])
def test_bitexact_vs_oracle_small(cuda_ok, chunk_words, planes, path):
    torch = cuda_ok
    geo = _small_geometry(chunk_words, planes)
    G, C = 96, 80
    cache, host, dp = _mk(torch, geo, G, C, path=path[0], piece=path[1], stages=path[2])
    rng = np.random.default_rng(chunk_words)
    pattern = orc.kv_pattern(7, geo.num_planes, G, geo.plane_chunk_bytes)
    cache.planes.copy_(torch.from_numpy(pattern))
    host.array[:] = 0xAB
    # a contiguous stretch (-> multi-block ops) inside otherwise random,
    # duplicate-free tables
    run_g, run_c = np.arange(50, 60), np.arange(30, 40)
    gpu_tab = np.concatenate([orc.random_block_table(rng, 5, G, used=run_g), run_g])
    gpu_tab = np.concatenate([gpu_tab, orc.random_block_table(rng, 25, G, used=gpu_tab)])
    cpu_tab = np.concatenate([orc.random_block_table(rng, 5, C, used=run_c), run_c])
    cpu_tab = np.concatenate([cpu_tab, orc.random_block_table(rng, 25, C, used=cpu_tab)])
    assert len(set(gpu_tab)) == len(set(cpu_tab)) == 40
    ops = orc.table_to_ops(gpu_tab, cpu_tab)
    assert ops[:, 0].max() > 1

    dp.swap("out", ops)
    torch.cuda.synchronize()
    want_host = np.full((C, geo.block_bytes), 0xAB, dtype=np.uint8)
    orc.apply_plan("out", pattern.copy(), want_host, ops)
    np.testing.assert_array_equal(host.array, want_host)

    # swap-in to a different table over a poisoned pool
    cache.planes.fill_(0xFF)
    new_gpu = orc.random_block_table(rng, 40, G)
    in_ops = orc.table_to_ops(new_gpu, cpu_tab)
    dp.swap("in", in_ops)
    torch.cuda.synchronize()
    want_planes = np.full_like(pattern, 0xFF)
    orc.apply_plan("in", want_planes, want_host, in_ops)
    np.testing.assert_array_equal(cache.planes.cpu().numpy(), want_planes)
    # and the logical content is the original one
    got = cache.planes.cpu().numpy()
    for k in range(40):
        np.testing.assert_array_equal(got[:, new_gpu[k]], pattern[:, gpu_tab[k]])
    host.close()


@pytest.mark.parametrize("path", ["lsu", "bulk"])
def test_split_single_and_many_ops(cuda_ok, path):
    """Baseline ablation ops (swap.py:170-179) and >2048-op plans (multi-launch)."""
    torch = cuda_ok
    geo = _small_geometry(64, 2)
    G = C = 5000
    cache, host, dp = _mk(torch, geo, G, C, path=path)
    rng = np.random.default_rng(3)
    pattern = orc.kv_pattern(11, geo.num_planes, G, geo.plane_chunk_bytes)
    cache.planes.copy_(torch.from_numpy(pattern))
    gpu_tab = orc.random_block_table(rng, 4500, G)
    cpu_tab = orc.random_block_table(rng, 4500, C)
    ops = orc.table_to_ops(gpu_tab, cpu_tab)
    assert len(ops) > 2048
    single = orc.split_single(ops)
    host.array[:] = 0
    dp.swap("out", single)
    torch.cuda.synchronize()
    want = np.zeros((C, geo.block_bytes), dtype=np.uint8)
    orc.apply_plan("out", pattern, want, ops)
    np.testing.assert_array_equal(host.array, want)
    host.close()


def test_empty_and_bad_ops(cuda_ok):
    torch = cuda_ok
    geo = _small_geometry(64, 2)
    cache, host, dp = _mk(torch, geo, 16, 16)
    before = dp.launches
    dp.swap("out", np.zeros((0, 3), dtype=np.int32))
    assert dp.launches == before  # nothing to move, nothing launched
    with pytest.raises(IndexError):
        dp.swap("out", [(4, 14, 0)])  # GPU side past the pool
    with pytest.raises(IndexError):
        dp.swap("in", [(4, 0, 13)])  # host side past the pool
    with pytest.raises(ValueError):
        dp.swap("out", [(0, 0, 0)])  # zero-block op
    with pytest.raises(KeyError):
        dp.swap("sideways", [(1, 0, 0)])
    with pytest.raises(ValueError):
        dp.set_path("out", "bulk", piece_bytes=100)  # not a 16-B multiple
    with pytest.raises(ValueError):
        dp.set_path("out", "bulk", piece_bytes=65536, stages=8)  # > 227 KiB smem
    host.close()


@pytest.mark.parametrize("slot_blocks,slots", [(1, 2), (3, 2), (7, 4), (0, 0)])
@pytest.mark.parametrize("chunk_words,planes", [(1028, 3), (4, 1), (256, 4)])
def test_staged_copy_engine_path_vs_oracle(cuda_ok, chunk_words, planes, slot_blocks, slots):
    """Staged path (kvs_memcpy_baseline mode 2): host runs through an HBM ring
    of `slots` slots of `slot_blocks` blocks, gather / scatter kernel on the
    handle's auxiliary stream.  Bit-exact vs the oracle for ops that span
    slots, host runs that continue across ops (one copy), several plans in a
    row (ring wrap); stream order on both sides: the swap-out sees KV written
    on its stream just before the call, and work queued on the stream after a
    swap-in sees every byte without a host sync in between."""
    torch = cuda_ok
    geo = _small_geometry(chunk_words, planes)
    G, C = 96, 80
    cache, host, dp = _mk(torch, geo, G, C)
    dp.set_staging(slot_blocks * geo.block_bytes, slots)
    rng = np.random.default_rng(chunk_words + 17 * slot_blocks)
    pattern = orc.kv_pattern(11, geo.num_planes, G, geo.plane_chunk_bytes)
    s = torch.cuda.Stream()
    launches0 = dp.launches
    for rep in range(3):
        host.array[:] = 0xAB
        # host blocks 20..28 in order under random GPU blocks: consecutive ops
        # whose host runs continue (one copy), then random pairs
        gpu_tab = orc.random_block_table(rng, 40, G)
        cpu_tab = np.concatenate([np.arange(20, 29), orc.random_block_table(
            rng, 31, C, used=np.arange(20, 29))])
        ops = orc.table_to_ops(gpu_tab, cpu_tab)
        with torch.cuda.stream(s):
            cache.planes.copy_(torch.from_numpy(pattern).to("cuda:0", non_blocking=False))
            cache.planes.add_(rep)  # written on s right before the swap-out
        dp.baseline("out", 2, ops, stream=s)
        s.synchronize()
        want = np.full((C, geo.block_bytes), 0xAB, dtype=np.uint8)
        orc.apply_plan("out", pattern + np.uint8(rep), want, ops)
        np.testing.assert_array_equal(host.array, want)
        with torch.cuda.stream(s):
            cache.planes.fill_(0x5A)
        new_gpu = orc.random_block_table(rng, sum(o[0] for o in ops), G)
        cpu_order = np.concatenate([np.arange(o[2], o[2] + o[0]) for o in ops])
        in_ops = orc.table_to_ops(new_gpu, cpu_order)
        dp.baseline("in", 2, in_ops, stream=s)
        with torch.cuda.stream(s):
            seen = cache.planes.clone()  # queued after the call, no host sync
        s.synchronize()
        want_planes = np.full_like(pattern, 0x5A)
        orc.apply_plan("in", want_planes, want, in_ops)
        np.testing.assert_array_equal(seen.cpu().numpy(), want_planes)
    assert dp.launches > launches0  # the gather / scatter kernels ran
    host.close()


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_copy_engine_baselines_match(cuda_ok, mode):
    """K3 per-block / per-run and the staged copy-engine path move the same bytes."""
    torch = cuda_ok
    geo = _small_geometry(256, 4)
    G, C = 128, 128
    cache, host, dp = _mk(torch, geo, G, C)
    rng = np.random.default_rng(mode)
    pattern = orc.kv_pattern(5, geo.num_planes, G, geo.plane_chunk_bytes)
    cache.planes.copy_(torch.from_numpy(pattern))
    ops = orc.random_runs(rng, 64, 8, G, C)
    s = torch.cuda.Stream()
    host.array[:] = 0
    dp.baseline("out", mode, ops, stream=s)
    s.synchronize()
    want = np.zeros((C, geo.block_bytes), dtype=np.uint8)
    orc.apply_plan("out", pattern, want, ops)
    np.testing.assert_array_equal(host.array, want)
    cache.planes.zero_()
    dp.baseline("in", mode, ops, stream=s)
    s.synchronize()
    want_planes = np.zeros_like(pattern)
    orc.apply_plan("in", want_planes, want, ops)
    np.testing.assert_array_equal(cache.planes.cpu().numpy(), want_planes)
    host.close()


@pytest.mark.parametrize("path", ["lsu", "bulk"])
def test_done_flag_orders_streams(cuda_ok, path):
    """kvs_swap's done flag + kvs_wait_flag: a consumer stream waits for the
    swap-out before reusing its source blocks (engine.py:712-719 dependency)."""
    torch = cuda_ok
    geo = _small_geometry(1024, 4)
    G = C = 512
    cache, host, dp = _mk(torch, geo, G, C, ctas={"out": 2}, path=path)
    pattern = orc.kv_pattern(9, geo.num_planes, G, geo.plane_chunk_bytes)
    cache.planes.copy_(torch.from_numpy(pattern))
    flag = torch.zeros(1, dtype=torch.int32, device="cuda:0")
    out_s, in_s = torch.cuda.Stream(), torch.cuda.Stream()
    ops = [(G, 0, 0)]
    for seq in (1, 2, 3):
        dp.swap("out", ops, stream=out_s, done_flag=flag.data_ptr(), seq=seq)
        dp.wait_flag(in_s, flag.data_ptr(), seq)
        with torch.cuda.stream(in_s):
            cache.planes.fill_(seq)  # overwrite the freed source blocks
        torch.cuda.synchronize()
        assert int(flag.item()) == seq
        if seq == 1:
            want = np.zeros((C, geo.block_bytes), dtype=np.uint8)
            orc.apply_plan("out", pattern, want, ops)
            np.testing.assert_array_equal(host.array, want)
        else:
            assert (host.array == seq - 1).all()
    host.close()


def _swap_path(dp, path, direction, ops, stream):
    """One plan through the kernel (LSU / TMA bulk) or the staged copy-engine path."""
    if path == "staged":
        dp.baseline(direction, 2, ops, stream=stream)
    else:
        dp.swap(direction, ops, stream=stream)


@pytest.mark.parametrize("path", ["lsu", "bulk", "staged"])
def test_config1_round_trip_llama3_8b(cuda_ok, path):
    """BASELINE config 1 at full size: 64 requests, LLaMA-3-8B KV shape
    (2 MiB blocks), footprints U{1..128}, fragmented random block tables,
    swap all out, poison HBM, swap all back into fresh tables."""
    torch = cuda_ok
    from paper_2411_18424_b200.geometry import LLAMA3_8B

    G = C = 8192
    cache, host, dp = _mk(torch, LLAMA3_8B, G, C, path="lsu" if path == "staged" else path)
    gen = torch.Generator(device="cuda:0").manual_seed(0)
    cache.planes.view(torch.int32).random_(generator=gen)
    rng = np.random.default_rng(0)
    foot = rng.integers(1, 129, size=64)
    total = int(foot.sum())
    gpu_tab = orc.random_block_table(rng, total, G)
    cpu_tab = orc.random_block_table(rng, total, C)
    bounds = np.concatenate([[0], np.cumsum(foot)])
    original = cache.planes[:, torch.from_numpy(gpu_tab).cuda()].clone()
    host.array[:] = 0xA5  # every host byte the plans do not own must stay this
    torch.cuda.synchronize()  # the KV fill runs on torch's stream, the swaps on s_out
    s_out, s_in = torch.cuda.Stream(), torch.cuda.Stream()
    out_plans = []
    for r in range(64):
        lo, hi = bounds[r], bounds[r + 1]
        out_plans.append(orc.table_to_ops(gpu_tab[lo:hi], cpu_tab[lo:hi]))
        _swap_path(dp, path, "out", out_plans[-1], s_out)
    torch.cuda.synchronize()
    # The whole host image against the oracle (TransferOp semantics,
    # bytes_oracle.apply_plan): the block the oracle's bijection maps each GPU
    # block to holds that block's planes in plane order, and no other host
    # byte changed.  A transposition applied symmetrically by both kernels
    # would survive the round trip below but not this.
    pairs = np.concatenate([orc.block_pairs(ops) for ops in out_plans])
    g_idx = torch.from_numpy(pairs[:, 0]).cuda()
    want = cache.planes.index_select(1, g_idx).permute(1, 0, 2).reshape(len(pairs), -1)
    got = host.tensor.index_select(0, torch.from_numpy(pairs[:, 1])).cuda()
    assert torch.equal(got, want)
    del got, want
    untouched = np.ones(C, dtype=bool)
    untouched[pairs[:, 1]] = False
    assert (host.array[untouched] == 0xA5).all()
    cache.planes.fill_(0xFF)
    torch.cuda.synchronize()  # the poison runs on torch's stream, the swaps on s_in
    new_tab = orc.random_block_table(rng, total, G)
    for r in range(64):
        lo, hi = bounds[r], bounds[r + 1]
        _swap_path(dp, path, "in", orc.table_to_ops(new_tab[lo:hi], cpu_tab[lo:hi]), s_in)
    torch.cuda.synchronize()
    back = cache.planes[:, torch.from_numpy(new_tab).cuda()]
    assert torch.equal(back, original)
    host.close()


@pytest.mark.parametrize("path", ["lsu", "bulk"])
@pytest.mark.parametrize("group", [0, 1, 4])
@pytest.mark.parametrize("direction", ["in", "out"])
def test_layered_swap_flags_each_plane(cuda_ok, direction, group, path):
    """kvs_swap_layered: plane-major order (in groups of `group` planes, 0 =
    auto; 6 planes / 4 leaves a partial last group), per-plane release flags;
    a consumer stream waiting on plane l's flag sees plane l's bytes complete."""
    torch = cuda_ok
    geo = _small_geometry(1028, 6)
    G = C = 600
    cache, host, dp = _mk(torch, geo, G, C, ctas={"out": 4, "in": 4}, path=path)
    dp.set_layer_group(group)
    rng = np.random.default_rng(21)
    pattern = orc.kv_pattern(3, geo.num_planes, G, geo.plane_chunk_bytes)
    gpu_tab = orc.random_block_table(rng, 500, G)
    cpu_tab = orc.random_block_table(rng, 500, C)
    ops = orc.table_to_ops(gpu_tab, cpu_tab)
    if direction == "in":
        host_img = np.zeros((C, geo.block_bytes), np.uint8)
        orc.apply_plan("out", pattern, host_img, ops)
        host.array[:] = host_img
        cache.planes.zero_()
    else:
        cache.planes.copy_(torch.from_numpy(pattern))
        host.array[:] = 0
    torch.cuda.synchronize()
    flags = torch.zeros(geo.num_planes, dtype=torch.int32, device="cuda:0")
    s_swap, s_use = torch.cuda.Stream(), torch.cuda.Stream()
    snaps = []
    dp.swap_layered(direction, ops, flags.data_ptr(), 1, stream=s_swap)
    if direction == "in":
        idx = torch.from_numpy(gpu_tab).cuda()
        for l in range(geo.num_planes):
            dp.wait_flag(s_use, flags.data_ptr() + 4 * l, 1)
            with torch.cuda.stream(s_use):
                snaps.append(cache.planes[l, idx].clone())  # "decode of layer l"
    torch.cuda.synchronize()
    assert flags.tolist() == [1] * geo.num_planes
    if direction == "in":
        for l in range(geo.num_planes):
            assert np.array_equal(snaps[l].cpu().numpy(), pattern[l, gpu_tab])
        want = np.zeros_like(pattern)
        orc.apply_plan("in", want, host.array.copy(), ops)
        np.testing.assert_array_equal(cache.planes.cpu().numpy(), want)
    else:
        want = np.zeros((C, geo.block_bytes), np.uint8)
        orc.apply_plan("out", pattern, want, ops)
        np.testing.assert_array_equal(host.array, want)
    # generation 2 on the same handle: counters carry over, flags advance
    dp.swap_layered(direction, ops, flags.data_ptr(), 2, stream=s_swap)
    torch.cuda.synchronize()
    assert flags.tolist() == [2] * geo.num_planes
    host.close()


@pytest.mark.parametrize("path", ["lsu", "bulk"])
def test_op_flags_signal_each_transfer_op(cuda_ok, path):
    """kvs_swap_ops: op i's flag <- seq once op i landed; a consumer waiting
    on one op's flag sees that op's bytes complete (op-granular conflicts).
    The TMA bulk path credits ops on its store side (after the stores
    complete), the LSU path per warp."""
    torch = cuda_ok
    geo = _small_geometry(1028, 4)
    G = C = 4096
    cache, host, dp = _mk(torch, geo, G, C, ctas={"out": 2}, path=path)
    pattern = orc.kv_pattern(13, geo.num_planes, G, geo.plane_chunk_bytes)
    cache.planes.copy_(torch.from_numpy(pattern))
    host.array[:] = 0
    torch.cuda.synchronize()
    rng = np.random.default_rng(5)
    ops = orc.random_runs(rng, 1600, 100, G, C)  # 16 ops of 100 blocks
    flags = torch.zeros(len(ops) + 3000, dtype=torch.int32, device="cuda:0")
    done = torch.zeros(1, dtype=torch.int32, device="cuda:0")
    s_swap, s_use = torch.cuda.Stream(), torch.cuda.Stream()
    dp.swap_ops("out", ops, flags.data_ptr(), 7, stream=s_swap, done_flag=done.data_ptr())
    k = 3
    dp.wait_flag(s_use, flags.data_ptr() + 4 * k, 7)
    b, g, c = (int(x) for x in ops[k])
    with torch.cuda.stream(s_use):
        cache.planes[:, g:g + b].fill_(0xEE)  # reuse op k's source blocks early
    torch.cuda.synchronize()
    assert flags[:len(ops)].tolist() == [7] * len(ops) and int(done.item()) == 7
    want = np.zeros((C, geo.block_bytes), np.uint8)
    orc.apply_plan("out", pattern, want, ops)
    np.testing.assert_array_equal(host.array, want)  # op k was read before the overwrite
    # > 2048 ops: flags of every launch slice
    many = orc.random_runs(rng, 2500, 1, G, C)
    dp.swap_ops("in", many, flags.data_ptr(), 8, stream=s_swap)
    torch.cuda.synchronize()
    assert (flags[:len(many)] == 8).all()
    host.close()


def test_executor_op_granular_conflict_wait(cuda_ok):
    """StreamExecutor: compute waits on the blocking op's flag, not the plan."""
    torch = cuda_ok
    from paper_2411_18424_b200.cpu_store import TransferOp
    from paper_2411_18424_b200.swap import StreamExecutor

    geo = _small_geometry(1028, 4)
    cache, host, dp = _mk(torch, geo, 1024, 1024)
    ex = StreamExecutor(dp)
    pattern = orc.kv_pattern(17, geo.num_planes, 1024, geo.plane_chunk_bytes)
    cache.planes.copy_(torch.from_numpy(pattern))
    torch.cuda.synchronize()
    ops = [TransferOp(64, 64 * i, 64 * i) for i in range(10)]
    ex.submit("out", ops)
    assert ex.compute_barrier([(64 * 2 + 5, 3)]) == 1  # overlaps op 2 only
    assert ex.op_waits == 1 and ex.plan_waits == 0
    with torch.cuda.stream(ex.compute):
        cache.planes[:, 133:136].fill_(0x11)
    ex.synchronize()
    want = np.zeros((1024, geo.block_bytes), np.uint8)
    orc.apply_plan("out", pattern, want, [(o.blocks, o.gpu_start, o.cpu_start) for o in ops])
    np.testing.assert_array_equal(host.array[:640], want[:640])
    host.close()


def test_registered_numa_host_pool(cuda_ok):
    """kvs_host_alloc(KVS_HOST_REGISTER): mmap + mbind(node 0) + cudaHostRegister."""
    torch = cuda_ok
    from paper_2411_18424_b200.dataplane import HostKVPool, PagedKVCache, SwapDataPlane

    geo = _small_geometry(1024, 2)
    cache = PagedKVCache(geo, 64, device="cuda:0")
    host = HostKVPool(64, geo.block_bytes, numa_node=0, register=True)
    dp = SwapDataPlane(cache, host)
    pattern = orc.kv_pattern(2, geo.num_planes, 64, geo.plane_chunk_bytes)
    cache.planes.copy_(torch.from_numpy(pattern))
    ops = [(10, 5, 40), (3, 50, 0)]
    dp.swap("out", ops)
    torch.cuda.synchronize()
    want = np.zeros((64, geo.block_bytes), np.uint8)
    orc.apply_plan("out", pattern, want, ops)
    np.testing.assert_array_equal(host.array[[*range(40, 50), 0, 1, 2]],
                                  want[[*range(40, 50), 0, 1, 2]])
    host.close()


@pytest.mark.parametrize("path", ["lsu", "bulk"])
def test_pacing_and_shared_budget(cuda_ok, path):
    """kvs_set_pace / kvs_set_budget: the rate is honoured and bytes stay exact."""
    torch = cuda_ok
    from paper_2411_18424_b200.geometry import LLAMA3_8B

    G = C = 1024
    cache, host, dp = _mk(torch, LLAMA3_8B, G, C, path=path)
    gen = torch.Generator(device="cuda:0").manual_seed(1)
    cache.planes.view(torch.int32).random_(generator=gen)
    torch.cuda.synchronize()  # the fill runs on torch's stream, the swaps on s1 / s2
    rng = np.random.default_rng(9)
    ops = orc.random_runs(rng, 256, 16, G // 2, C // 2)  # 512 MiB
    ops_in = ops.copy()
    ops_in[:, 1:] += G // 2
    nbytes = 256 * LLAMA3_8B.block_bytes
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn, stream):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        return e0, e1

    dp.set_pace("out", 20.0)
    e = timed(lambda: dp.swap("out", ops, stream=s1), s1)
    torch.cuda.synchronize()
    gbs = nbytes / (e[0].elapsed_time(e[1]) * 1e-3) / 1e9
    assert 12.0 < gbs < 21.0, gbs  # paced to 20 GB/s (globaltimer slots)
    want = np.zeros((C, LLAMA3_8B.block_bytes), np.uint8)
    orc.apply_plan("out", cache.planes.cpu().numpy(), want, ops)
    host_rows = np.concatenate([np.arange(c, c + b) for b, g, c in ops])
    np.testing.assert_array_equal(host.array[host_rows], want[host_rows])
    # shared budget: both directions together <= 30 GB/s
    dp.set_pace("out", 0.0)
    dp.set_budget(30.0)
    ref = torch.cuda.Event(enable_timing=True)
    ref.record()
    torch.cuda.synchronize()  # both streams start after `ref`: times are relative to it
    eo = timed(lambda: dp.swap("out", ops, stream=s1), s1)
    ei = timed(lambda: dp.swap("in", ops_in, stream=s2), s2)
    torch.cuda.synchronize()
    # union of the two kernels' lifetimes, not the longer one alone (they
    # need not start together)
    t0 = min(ref.elapsed_time(eo[0]), ref.elapsed_time(ei[0]))
    t1 = max(ref.elapsed_time(eo[1]), ref.elapsed_time(ei[1]))
    total = 2 * nbytes / ((t1 - t0) * 1e-3) / 1e9
    assert total < 33.0, total  # shared 30 GB/s budget (+ idle burst credit)
    dp.set_budget(0.0)
    host.close()


@pytest.mark.parametrize("model,tp", [("qwen2.5-32b", 2), ("qwen2.5-32b", 4),
                                      ("qwen2.5-32b", 8), ("llama3-70b", 8)])
@pytest.mark.parametrize("path", ["lsu", "staged"])
def test_tp_shard_shapes_vs_oracle(cuda_ok, model, tp, path):
    """BASELINE configs 4-5: per-rank KV shards (32 / 16 / 8 KiB chunks, 64-80
    planes), C5-like long runs; swap-out byte-exact vs the oracle, then
    swap-in to a new table == the oracle's restatement of the same ops, on
    the kernel and on the staged copy-engine path."""
    torch = cuda_ok
    from paper_2411_18424_b200.geometry import PRESETS

    geo = PRESETS[model].with_tp(tp)
    G = C = 768
    cache, host, dp = _mk(torch, geo, G, C)
    rng = np.random.default_rng(tp)
    pattern = orc.kv_pattern(tp, geo.num_planes, G, geo.plane_chunk_bytes)
    cache.planes.copy_(torch.from_numpy(pattern))
    ops = orc.random_runs(rng, 600, 145, G, C)  # C5: mean 145 blocks per op
    host.array[:] = 0
    _swap_path(dp, path, "out", ops, None)
    torch.cuda.synchronize()
    want = np.zeros((C, geo.block_bytes), dtype=np.uint8)
    orc.apply_plan("out", pattern, want, ops)
    np.testing.assert_array_equal(host.array, want)
    cache.planes.fill_(0xA5)
    torch.cuda.synchronize()
    in_ops = orc.random_runs(rng, 600, 37, G, C)
    _swap_path(dp, path, "in", in_ops, None)
    torch.cuda.synchronize()
    want_planes = np.full_like(pattern, 0xA5)
    orc.apply_plan("in", want_planes, want, in_ops)
    assert np.array_equal(cache.planes.cpu().numpy(), want_planes)
    host.close()


def test_sm_partition_streams_move_exact_bytes(cuda_ok):
    """kvs_sm_partition (green contexts): swap kernels launched on the swap
    side's streams, a torch kernel on the compute side; bytes exact."""
    torch = cuda_ok
    from paper_2411_18424_b200.swap import partition_streams

    (s_out, s_in), comp, sms = partition_streams(torch.device("cuda:0"), 8)
    props = torch.cuda.get_device_properties(0)
    assert sms[0] >= 8 and sms[0] + sms[1] == props.multi_processor_count
    geo = _small_geometry(1024, 4)
    G = C = 256
    cache, host, dp = _mk(torch, geo, G, C)
    pattern = orc.kv_pattern(21, geo.num_planes, G, geo.plane_chunk_bytes)
    cache.planes.copy_(torch.from_numpy(pattern))
    torch.cuda.synchronize()
    rng = np.random.default_rng(21)
    ops = orc.random_runs(rng, 120, 8, G, C)
    host.array[:] = 0
    dp.swap("out", ops, stream=s_out)
    s_out.synchronize()
    want = np.zeros((C, geo.block_bytes), dtype=np.uint8)
    orc.apply_plan("out", pattern, want, ops)
    np.testing.assert_array_equal(host.array, want)
    with torch.cuda.stream(comp):
        cache.planes.fill_(0x3C)  # compute side: a torch kernel on the other SM group
    comp.synchronize()
    dp.swap("in", ops, stream=s_in)
    s_in.synchronize()
    want_planes = np.full_like(pattern, 0x3C)
    orc.apply_plan("in", want_planes, want, ops)
    assert np.array_equal(cache.planes.cpu().numpy(), want_planes)
    host.close()


@pytest.mark.parametrize("n_ops_big", [False, True])
def test_signaled_swap_op_plane_and_done_flags(cuda_ok, n_ops_big):
    """kvs_swap_signaled: per-op + per-plane + whole-plan words from one call
    (plane-major order, > 2048 ops -> several launches); a consumer waiting on
    plane l sees plane l complete; bytes exact vs the oracle."""
    torch = cuda_ok
    geo = _small_geometry(1028, 5)
    G = C = 3000
    cache, host, dp = _mk(torch, geo, G, C, ctas={"out": 4, "in": 4})
    rng = np.random.default_rng(33)
    pattern = orc.kv_pattern(8, geo.num_planes, G, geo.plane_chunk_bytes)
    n = 2600 if n_ops_big else 400
    gpu_tab = orc.random_block_table(rng, n, G)
    cpu_tab = orc.random_block_table(rng, n, C)
    ops = orc.table_to_ops(gpu_tab, cpu_tab)
    assert (len(ops) > 2048) == n_ops_big
    host_img = np.zeros((C, geo.block_bytes), np.uint8)
    orc.apply_plan("out", pattern, host_img, ops)
    host.array[:] = host_img
    cache.planes.zero_()
    torch.cuda.synchronize()
    words = torch.zeros(len(ops) + geo.num_planes + 1, dtype=torch.int32, device="cuda:0")
    base = words.data_ptr()
    s_swap, s_use = torch.cuda.Stream(), torch.cuda.Stream()
    dp.swap_signaled("in", ops, 5, op_flags=base, plane_flags=base + 4 * len(ops),
                     done_flag=base + 4 * (len(ops) + geo.num_planes), stream=s_swap)
    idx = torch.from_numpy(gpu_tab).cuda()
    snaps = []
    for l in range(geo.num_planes):
        dp.wait_flag(s_use, base + 4 * (len(ops) + l), 5)
        with torch.cuda.stream(s_use):
            snaps.append(cache.planes[l, idx].clone())
    torch.cuda.synchronize()
    assert words.tolist() == [5] * words.numel()
    for l in range(geo.num_planes):
        assert np.array_equal(snaps[l].cpu().numpy(), pattern[l, gpu_tab])
    want = np.zeros_like(pattern)
    orc.apply_plan("in", want, host_img, ops)
    np.testing.assert_array_equal(cache.planes.cpu().numpy(), want)
    with pytest.raises(ValueError):  # reserved field must be zero
        from paper_2411_18424_b200 import _lib
        import ctypes
        bad = _lib.KvsSignals(None, None, None, 1, 7)
        _lib.check(dp.lib.kvs_swap_signaled(dp.handle, 1, None, 0, 0, ctypes.byref(bad)))
    host.close()


def test_split_kv_layout_vs_oracle(cuda_ok):
    """vLLM-v0 style split K/V caches ([2, num_blocks, ...] per layer) are two
    planes per layer; same block bytes as the fused layout, byte-exact."""
    torch = cuda_ok
    from paper_2411_18424_b200.geometry import KVGeometry

    fused = KVGeometry("s", num_layers=4, num_kv_heads=2, head_dim=64)
    geo = KVGeometry("s", num_layers=4, num_kv_heads=2, head_dim=64, split_kv=True)
    assert geo.num_planes == 2 * fused.num_planes and geo.block_bytes == fused.block_bytes
    G = C = 200
    cache, host, dp = _mk(torch, geo, G, C)
    rng = np.random.default_rng(17)
    pattern = orc.kv_pattern(17, geo.num_planes, G, geo.plane_chunk_bytes)
    cache.planes.copy_(torch.from_numpy(pattern))
    torch.cuda.synchronize()
    ops = orc.table_to_ops(orc.random_block_table(rng, 150, G), orc.random_block_table(rng, 150, C))
    host.array[:] = 0
    dp.swap("out", ops)
    torch.cuda.synchronize()
    want = np.zeros((C, geo.block_bytes), np.uint8)
    orc.apply_plan("out", pattern, want, ops)
    np.testing.assert_array_equal(host.array, want)
    cache.planes.zero_()
    torch.cuda.synchronize()
    dp.swap("in", ops)
    torch.cuda.synchronize()
    back = np.zeros_like(pattern)
    orc.apply_plan("in", back, want, ops)
    np.testing.assert_array_equal(cache.planes.cpu().numpy(), back)
    host.close()


def test_executor_throughput_policy_bulk_round_trip(cuda_ok):
    """The throughput policy runs both directions on the TMA bulk kernel with
    plan-level waits: a swap-in reading host blocks a queued swap-out writes
    (RAW across streams) still sees the swapped-out bytes."""
    torch = cuda_ok
    from paper_2411_18424_b200.cpu_store import TransferOp
    from paper_2411_18424_b200.swap import StreamExecutor

    geo = _small_geometry(1028, 4)
    cache, host, dp = _mk(torch, geo, 1024, 1024)
    ex = StreamExecutor(dp, duplex_policy="throughput")
    assert not ex.op_granular
    pattern = orc.kv_pattern(29, geo.num_planes, 1024, geo.plane_chunk_bytes)
    cache.planes.copy_(torch.from_numpy(pattern))
    torch.cuda.synchronize()
    out_ops = [TransferOp(40, 40 * i, 100 + 40 * i) for i in range(8)]
    in_ops = [TransferOp(40, 600 + 40 * i, 100 + 40 * i) for i in range(8)]
    l0 = dp.launches
    ex.submit("out", out_ops)
    rec = ex.submit("in", in_ops)  # must wait for the out plan (RAW on host blocks)
    assert rec.deps == 1 and ex.plan_waits == 1
    ex.synchronize()
    assert dp.launches - l0 == 2
    want = pattern.copy()
    host_img = np.zeros((1024, geo.block_bytes), np.uint8)
    orc.apply_plan("out", pattern, host_img, [(o.blocks, o.gpu_start, o.cpu_start) for o in out_ops])
    orc.apply_plan("in", want, host_img, [(o.blocks, o.gpu_start, o.cpu_start) for o in in_ops])
    np.testing.assert_array_equal(cache.planes.cpu().numpy(), want)
    ex.set_duplex_policy("latency")
    assert ex.op_granular
    host.close()


def test_kv_image_export_import_through_the_kernels(cuda_ok, tmp_path):
    """Swap-out with the kernel into pinned host memory, export the request's
    host image to a file, import it into another rank's pool at other host
    blocks, swap it in with the kernel: byte-exact."""
    torch = cuda_ok
    from paper_2411_18424_b200.cpu_store import CpuStore
    from paper_2411_18424_b200.geometry import LLAMA3_8B
    from paper_2411_18424_b200.kvimage import export_image, import_image

    geo = LLAMA3_8B.with_tp(4)  # 512 KiB blocks
    G = C = 128
    cache, host, dp = _mk(torch, geo, G, C)
    cache.planes.view(torch.int32).random_(generator=torch.Generator(device="cuda:0").manual_seed(3))
    torch.cuda.synchronize()
    store = CpuStore(C)
    gpu_ext = [(10, 20), (64, 13)]
    plan = store.plan_swap_out(7, 33, gpu_ext)
    dp.swap("out", plan.all_ops())
    torch.cuda.synchronize()
    path = str(tmp_path / "req7.kvimg")
    export_image(store, host.array, 7, geo, path)

    cache2, host2, dp2 = _mk(torch, geo, G, C)
    store2 = CpuStore(C)
    store2.plan_swap_out(1, 40, [(0, 40)])  # occupy the front of the second pool
    import_image(path, store2, host2.array, 7, geo)
    new_ext = [(90, 33)]
    dp2.swap("in", store2.plan_swap_in(7, new_ext).all_ops())
    torch.cuda.synchronize()
    src = torch.cat([cache.planes[:, s:s + n] for s, n in gpu_ext], dim=1)
    assert torch.equal(cache2.planes[:, 90:123], src)
    host.close()
    host2.close()


def test_budget_share_reserves_a_rate_for_one_direction(cuda_ok):
    """kvs_set_budget_share: with a 20 GB/s budget of which swap-in reserves
    15, a concurrent saturating swap-out leaves swap-in >= its share (FCFS
    would split the budget); bytes stay exact both ways."""
    torch = cuda_ok
    from paper_2411_18424_b200.geometry import LLAMA3_8B

    G = C = 1024
    cache, host, dp = _mk(torch, LLAMA3_8B, G, C)
    cache.planes.view(torch.int32).random_()
    host.array[:] = 0x3C
    torch.cuda.synchronize()
    out_ops = [(256, 0, 0)]       # 512 MiB out of GPU [0, 256) into host [0, 256)
    in_ops = [(128, 512, 512)]    # 256 MiB into GPU [512, 640) from host [512, 640)
    src = cache.planes[:, 0:256].clone()
    dp.set_budget(20.0)
    dp.set_budget_share("in", 15.0)
    s_out, s_in = torch.cuda.Stream(), torch.cuda.Stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record(s_out)
    dp.swap("out", out_ops, stream=s_out)
    ev[1].record(s_out)
    ev[2].record(s_in)
    dp.swap("in", in_ops, stream=s_in)
    ev[3].record(s_in)
    torch.cuda.synchronize()
    in_gbs = 128 * LLAMA3_8B.block_bytes / (ev[2].elapsed_time(ev[3]) * 1e-3) / 1e9
    out_ms = ev[0].elapsed_time(ev[1])
    if not under_sanitizer():  # rates mean nothing under compute-sanitizer
        assert in_gbs >= 0.85 * 15.0, in_gbs
        # the budget still binds the pair: out + in together stay near 20 GB/s
        total = (256 + 128) * LLAMA3_8B.block_bytes / (
            max(out_ms, ev[0].elapsed_time(ev[3])) * 1e-3) / 1e9
        assert total <= 1.15 * 20.0, total
    got = host.tensor[0:256].cuda().view(256, LLAMA3_8B.num_planes, -1).permute(1, 0, 2)
    assert torch.equal(got, src)
    assert (cache.planes[:, 512:640].cpu().numpy() == 0x3C).all()
    dp.set_budget(0.0)
    dp.set_budget_share("in", 0.0)
    host.close()
