"""The exported host KV image (paper_2411_18424_b200.kvimage): a request
swapped out on one store, exported, imported into another store at other
host blocks, and swapped in to another GPU table comes back byte-exact; bad
images are rejected.  Host-side only (numpy pools, oracle byte restatement)."""

import io

import numpy as np
import pytest

from oracle import bytes_oracle as orc
from paper_2411_18424_b200.cpu_store import CpuStore
from paper_2411_18424_b200.native_ctrl import NativeCpuStore
from paper_2411_18424_b200.geometry import KVGeometry
from paper_2411_18424_b200.kvimage import KVImageError, export_image, import_image

GEO = KVGeometry("img", num_layers=3, num_kv_heads=2, head_dim=8)  # 1 KiB chunks


@pytest.fixture(params=["python", "native"])
def Store(request):
    """Both control planes: the image round trip must not depend on it."""
    return CpuStore if request.param == "python" else NativeCpuStore


def _table(extents):
    return np.concatenate([np.arange(s, s + n) for s, n in extents])


def test_export_import_round_trip_is_byte_exact(Store):
    G, C = 96, 128
    planes = orc.kv_pattern(3, GEO.num_planes, G, GEO.plane_chunk_bytes)
    store, pool = Store(C), np.zeros((C, GEO.block_bytes), np.uint8)
    gpu_ext = [(30, 12), (70, 9)]
    plan = store.plan_swap_out(5, 21, gpu_ext, tokens=21 * 16 - 5)
    orc.apply_plan("out", planes, pool, [(o.blocks, o.gpu_start, o.cpu_start)
                                         for o in plan.all_ops()])
    buf = io.BytesIO()
    hdr = export_image(store, pool, 5, GEO, buf)
    assert hdr["blocks"] == 21 and hdr["tokens"] == 21 * 16 - 5

    # another rank: some host blocks already taken, so the image lands elsewhere
    store2, pool2 = Store(C), np.zeros((C, GEO.block_bytes), np.uint8)
    store2.plan_swap_out(9, 17, [(0, 17)])
    buf.seek(0)
    copy = import_image(buf, store2, pool2, 11, GEO)
    assert copy.valid_prefix_blocks() == 21 and copy.saved_tokens == hdr["tokens"]
    assert store2.pool.owned_blocks(11) == 21

    new_ext = [(5, 4), (50, 17)]
    plan_in = store2.plan_swap_in(11, new_ext)
    restored = np.zeros_like(planes)
    orc.apply_plan("in", restored, pool2, [(o.blocks, o.gpu_start, o.cpu_start)
                                           for o in plan_in.all_ops()])
    np.testing.assert_array_equal(restored[:, _table(new_ext)], planes[:, _table(gpu_ext)])


def test_corrupt_truncated_and_foreign_images_are_rejected(Store):
    G, C = 32, 32
    planes = orc.kv_pattern(4, GEO.num_planes, G, GEO.plane_chunk_bytes)
    store, pool = Store(C), np.zeros((C, GEO.block_bytes), np.uint8)
    plan = store.plan_swap_out(1, 6, [(2, 6)])
    orc.apply_plan("out", planes, pool, [(o.blocks, o.gpu_start, o.cpu_start) for o in plan.ops])
    buf = io.BytesIO()
    export_image(store, pool, 1, GEO, buf)
    raw = bytearray(buf.getvalue())

    flipped = bytearray(raw)
    flipped[-100] ^= 0x40
    with pytest.raises(KVImageError, match="corrupt"):
        import_image(io.BytesIO(bytes(flipped)), Store(C), pool.copy(), 1, GEO)
    with pytest.raises(KVImageError, match="truncated"):
        import_image(io.BytesIO(bytes(raw[:-10])), Store(C), pool.copy(), 1, GEO)
    with pytest.raises(KVImageError, match="magic"):
        import_image(io.BytesIO(b"NOTIMAGE" + bytes(raw[8:])), Store(C), pool.copy(), 1, GEO)
    other = KVGeometry("img", num_layers=3, num_kv_heads=2, head_dim=8, tp=2)
    with pytest.raises(KVImageError, match="geometry"):
        import_image(io.BytesIO(bytes(raw)), Store(C), np.zeros((C, other.block_bytes),
                                                                   np.uint8), 1, other)


def test_contaminated_copy_exports_only_the_tokens_its_prefix_holds(Store):
    """the header's token count is clamped to the exported blocks,
    so a resumer never skips recompute it owes (plan_swap_in_prefix rule)."""
    C = 40
    store, pool = Store(C), np.zeros((C, GEO.block_bytes), np.uint8)
    store.set_rank(1, 5)
    store.plan_swap_out(1, 10, [(0, 10)], tokens=160)
    store.plan_swap_out(1, 30, [(0, 30)], tokens=30 * 16 - 3)
    store.evict_for(0, 15)  # a better-ranked request takes the 20-block tail segment
    assert store.copy_of(1).valid_prefix_blocks() == 10
    buf = io.BytesIO()
    hdr = export_image(store, pool, 1, GEO, buf)
    assert hdr["blocks"] == 10 and hdr["tokens"] == 10 * 16
    buf.seek(0)
    copy = import_image(buf, Store(C), pool.copy(), 3, GEO)
    assert copy.saved_tokens == 160 and copy.valid_prefix_blocks() == 10


def test_unranked_import_never_evicts_and_ranked_import_does(Store):
    from paper_2411_18424_b200.cpu_store import CpuOutOfMemoryError

    C = 32
    store, pool = Store(C), np.zeros((C, GEO.block_bytes), np.uint8)
    store.plan_swap_out(1, 12, [(0, 12)])
    buf = io.BytesIO()
    export_image(store, pool, 1, GEO, buf)
    raw = buf.getvalue()

    full = Store(C)
    full.set_rank(9, 3)
    full.plan_swap_out(9, 25, [(0, 25)])  # 7 free blocks left
    with pytest.raises(CpuOutOfMemoryError):
        import_image(io.BytesIO(raw), full, pool.copy(), 4, GEO)
    assert full.copy_of(9).fully_valid  # nobody was contaminated
    copy = import_image(io.BytesIO(raw), full, pool.copy(), 4, GEO, rank=0)
    assert copy.valid_prefix_blocks() == 12
    assert not full.copy_of(9).fully_valid  # the lower-priority copy paid


class _FenceSpy:
    def __init__(self):
        self.calls = []

    def host_fence(self, rows):
        self.calls.append(list(rows))
        return 0


def test_export_and_import_fence_their_pool_rows_on_the_executor(Store):
    """CPU reads/writes of pool rows wait for in-flight transfers
    over those rows (StreamExecutor.host_fence)."""
    C = 64
    store, pool = Store(C), np.zeros((C, GEO.block_bytes), np.uint8)
    plan = store.plan_swap_out(2, 9, [(4, 9)])
    spy = _FenceSpy()
    buf = io.BytesIO()
    export_image(store, pool, 2, GEO, buf, executor=spy)
    cpu = [(o.cpu_start, o.blocks) for o in plan.ops]
    assert spy.calls == [cpu]
    buf.seek(0)
    store2 = Store(C)
    store2.plan_swap_out(5, 3, [(0, 3)])
    copy = import_image(buf, store2, np.zeros_like(pool), 6, GEO, executor=spy)
    placed = [(store2.pool.group(s.group_id).start, s.length) for s in copy.segments]
    assert spy.calls[1] == placed
