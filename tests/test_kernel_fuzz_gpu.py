"""Randomized byte parity of every kernel entry point against the oracle:
random geometries (1-7 planes, chunks from 16 B to 80 KiB, ragged against
the 4 KiB piece), random fragmented plans (1-2600 ops: multi-launch), both
directions, LSU and TMA-bulk paths, plain / op-flagged / layered (random
plane groups) / signaled launches, random launch shapes, and the staged
copy-engine path with random staging rings."""

import os

import numpy as np
import pytest

from oracle import bytes_oracle as orc

pytestmark = pytest.mark.gpu
CASES = int(os.environ.get("KVS_FUZZ_CASES", "24"))


@pytest.mark.parametrize("case", range(CASES))
def test_kernel_entry_points_match_oracle(cuda_ok, case):
    torch = cuda_ok
    from paper_2411_18424_b200.dataplane import HostKVPool, PagedKVCache, SwapDataPlane
    from paper_2411_18424_b200.geometry import KVGeometry

    rng = np.random.default_rng([7, case])
    planes = int(rng.integers(1, 8))
    words = int(rng.choice([1, 3, 4, 64, 257, 1024, 1028, 4100, 5120]))  # chunk = 16 * words
    geo = KVGeometry("fz", num_layers=planes, num_kv_heads=1, head_dim=4 * words, block_tokens=1)
    assert geo.plane_chunk_bytes == 16 * words
    G = C = int(rng.integers(64, 3000)) if geo.plane_chunk_bytes <= 4096 else 400
    cache = PagedKVCache(geo, G, device="cuda:0")
    host = HostKVPool(C, geo.block_bytes)
    dp = SwapDataPlane(cache, host)
    path = str(rng.choice(["lsu", "bulk"]))
    piece = int(rng.choice([0, 4096, 16384])) if path == "bulk" else 0
    dp.set_path("out", path, piece, int(rng.integers(2, 6)) if path == "bulk" else 0)
    dp.set_path("in", path, piece, int(rng.integers(2, 6)) if path == "bulk" else 0)
    for d in ("out", "in"):
        dp.set_launch(d, int(rng.choice([1, 3, 8, 37, 148])),
                      32 * int(rng.choice([1, 4, 8, 16])) if path == "lsu" else 0)
    dp.set_layer_group(int(rng.integers(0, planes + 1)))
    pattern = orc.kv_pattern(case, planes, G, geo.plane_chunk_bytes)
    cache.planes.copy_(torch.from_numpy(pattern))
    host.array[:] = 0
    torch.cuda.synchronize()
    n = int(rng.integers(1, min(G, C) - 1))
    gpu_tab = orc.random_block_table(rng, n, G)
    cpu_tab = orc.random_block_table(rng, n, C)
    ops = orc.table_to_ops(gpu_tab, cpu_tab)
    flags = torch.zeros(len(ops) + planes + 1, dtype=torch.int32, device="cuda:0")
    fp = flags.data_ptr()
    kind = str(rng.choice(["plain", "ops", "layered", "signaled", "staged"]))
    if kind == "staged":  # random ring: 1..40 blocks per slot, 2..5 slots
        dp.set_staging(int(rng.integers(1, 41)) * geo.block_bytes, int(rng.integers(2, 6)))

    def run(direction, seq):
        if kind == "plain":
            dp.swap(direction, ops)
        elif kind == "staged":
            dp.baseline(direction, 2, ops)
        elif kind == "ops":
            dp.swap_ops(direction, ops, fp, seq)
        elif kind == "layered":
            dp.swap_layered(direction, ops, fp + 4 * len(ops), seq)
        else:
            dp.swap_signaled(direction, ops, seq, op_flags=fp, plane_flags=fp + 4 * len(ops),
                             done_flag=fp + 4 * (len(ops) + planes))
        torch.cuda.synchronize()

    run("out", 1)
    want = np.zeros((C, geo.block_bytes), np.uint8)
    orc.apply_plan("out", pattern, want, ops)
    np.testing.assert_array_equal(host.array, want)
    cache.planes.fill_(0x5A)
    torch.cuda.synchronize()
    run("in", 2)
    back = np.full_like(pattern, 0x5A)
    orc.apply_plan("in", back, want, ops)
    np.testing.assert_array_equal(cache.planes.cpu().numpy(), back)
    f = flags.cpu().numpy()
    if kind in ("ops", "signaled"):
        assert (f[:len(ops)] == 2).all()
    if kind in ("layered", "signaled"):
        assert (f[len(ops):len(ops) + planes] == 2).all()
    if kind == "signaled":
        assert f[len(ops) + planes] == 2
    host.close()
