"""The decode step as a CUDA graph (kvs_graph_*, live.DecodeGraph): captured
attention (KV check) and weight-stream kernels run with each iteration's
parameters after an in-place update; plane-flag waits captured in the graph
hold the step until the flag is published; timing marks are read back."""

import time

import numpy as np
import pytest
import torch

from paper_2411_18424_b200.dataplane import HostKVPool, PagedKVCache, SwapDataPlane
from paper_2411_18424_b200.geometry import KVGeometry
from paper_2411_18424_b200.live import DecodeEmulator, DecodeGraph

from conftest import under_sanitizer  # noqa: E402

pytestmark = pytest.mark.gpu

GEO = KVGeometry("tiny-kv", num_layers=4, num_kv_heads=2, head_dim=8)  # 1 KiB chunks


def _setup():
    cache = PagedKVCache(GEO, 64, device="cuda:0")
    host = HostKVPool(16, GEO.block_bytes)
    dp = SwapDataPlane(cache, host)
    return cache, host, dp


def test_graph_updates_in_place_and_runs_each_iterations_parameters(cuda_ok):
    cache, host, dp = _setup()
    dec = DecodeEmulator("cuda:0", weight_bytes=64 << 20)
    bad = torch.zeros(1, dtype=torch.int32, device="cuda:0")
    g = DecodeGraph("cuda:0", marks=2 * GEO.num_planes)
    comp = torch.cuda.Stream()
    # KV of two requests written on the stream (the ordinary path)
    segs = np.array([[3, 0, 40, 5], [7, 0, 17, 20]], dtype=np.int64)
    dp.kv_tokens(0, segs, stream=comp)
    comp.synchronize()
    for it in range(4):
        # each iteration reads a different prefix of the KV (different grid)
        rd = segs.copy()
        rd[:, 2] = [40 - 7 * it, 17 - 3 * it]
        st = g.begin()
        for layer in range(GEO.num_planes):
            g.mark(2 * layer)
            dp.kv_tokens(1, rd, stream=st, mismatch_ptr=bad.data_ptr(), planes=(layer, layer + 1))
            dec.launch(st, (1 + it) << 20)
            g.mark(2 * layer + 1)
        how = g.end()
        assert how == (2 if it == 0 else 1)  # instantiated once, then updated in place
        g.launch(comp)
        comp.synchronize()
        assert int(bad.item()) == 0
        assert all(g.elapsed(2 * l, 2 * l + 1) > 0 for l in range(GEO.num_planes))
    # a corrupted KV word (plane 0, block 5, token 1's K row) is seen by the graph
    cache.planes[0, 5, 32] += 1
    st = g.begin()
    dp.kv_tokens(1, segs, stream=st, mismatch_ptr=bad.data_ptr(), planes=(0, 1))
    g.end()
    g.launch(comp)
    comp.synchronize()
    assert int(bad.item()) > 0
    assert g.stats()["launches"] == 5
    g.close()
    host.close()


def test_plane_flag_waits_are_graph_nodes(cuda_ok):
    """The producer of the flag is queued first (as in the live engine, where
    the swap-in is dispatched before the step that waits for its planes): a
    stream wait parks its hardware queue, so a producer queued after it on a
    queue it shares could never run."""
    cache, host, dp = _setup()
    flags = torch.zeros(4, dtype=torch.int32, device="cuda:0")
    g = DecodeGraph("cuda:0", marks=2)
    comp, side = torch.cuda.Stream(), torch.cuda.Stream()
    segs = np.array([[1, 0, 16, 9]], dtype=np.int64)
    st = g.begin()
    dp.wait_flag(st, flags.data_ptr() + 4 * 2, 5)  # waits for flags[2] >= 5
    g.mark(0)
    dp.kv_tokens(0, segs, stream=st)  # writes request 1's KV after the wait
    g.mark(1)
    g.end()
    cache.planes.zero_()
    torch.cuda.synchronize()
    with torch.cuda.stream(side):
        torch.cuda._sleep(300_000_000)  # ~0.15 s of GPU cycles, then publish the flag
        flags[2:3].fill_(5)
    g.launch(comp)
    early = comp.query()
    deadline = time.time() + 20
    while not comp.query():
        assert time.time() < deadline, "the graph never left its flag wait"
        time.sleep(0.002)
    if not under_sanitizer():  # compute-sanitizer skews the timing
        assert not early  # it was parked on the flag
    torch.cuda.synchronize()
    assert int(cache.planes.view(torch.int32).abs().sum().item()) > 0
    assert g.elapsed(0, 1) > 0
    g.close()
    host.close()


def test_one_call_step_capture_matches_and_waits_per_layer(cuda_ok):
    """kvs_graph_decode_step (DecodeGraph.capture_step): the whole step in one
    native call.  It reads the same KV as the per-call capture (a corrupted
    word in one plane is counted), streams the weights, and layer l of the
    step waits for plane flag l of every dependency: with the flags of
    planes >= 2 unpublished, the marks of layers 0-1 complete while the step
    is still parked."""
    cache, host, dp = _setup()
    dec = DecodeEmulator("cuda:0", weight_bytes=64 << 20)
    bad = torch.zeros(1, dtype=torch.int32, device="cuda:0")
    g = DecodeGraph("cuda:0", marks=2 * GEO.num_planes)
    comp, side = torch.cuda.Stream(), torch.cuda.Stream()
    segs = np.array([[3, 0, 40, 5], [7, 0, 17, 20]], dtype=np.int64)
    dp.kv_tokens(0, segs, stream=comp)
    comp.synchronize()
    for it in range(3):
        how = g.capture_step(dp, dec, segs, bad.data_ptr(), (1 + it) << 20, marks=True)
        assert how == (2 if it == 0 else 1)
        g.launch(comp)
        comp.synchronize()
        assert int(bad.item()) == 0
        assert all(g.elapsed(2 * l, 2 * l + 1) > 0 for l in range(GEO.num_planes))
    cache.planes[2, 20, 0] += 1  # request 7's first K word in plane 2
    g.capture_step(dp, dec, segs, bad.data_ptr(), 1 << 20)
    g.launch(comp)
    comp.synchronize()
    assert int(bad.item()) == 1
    # per-layer waits on two dependencies' plane flags
    flags = torch.zeros(2, GEO.num_planes, dtype=torch.int32, device="cuda:0")
    flags[:, :2] = 9
    deps = [(flags[0].data_ptr(), 9), (flags[1].data_ptr(), 9)]
    bad.zero_()
    cache.planes[2, 20, 0] -= 1
    torch.cuda.synchronize()
    g.capture_step(dp, dec, segs, bad.data_ptr(), 1 << 20, deps=deps, marks=True)
    with torch.cuda.stream(side):
        torch.cuda._sleep(300_000_000)
        flags[:, 2:].fill_(9)
    g.launch(comp)
    time.sleep(0.05)
    if not under_sanitizer():
        assert not comp.query()  # parked at layer 2's waits
    deadline = time.time() + 20
    while not comp.query():
        assert time.time() < deadline, "the step never left its plane-flag waits"
        time.sleep(0.002)
    assert int(bad.item()) == 0
    assert all(g.elapsed(2 * l, 2 * l + 1) > 0 for l in range(GEO.num_planes))
    g.close()
    host.close()


def test_failed_step_capture_leaves_no_runnable_graph(cuda_ok):
    """A capture that fails midway (a KV segment past the pool) raises, drops
    the partial step and the executable graph (a launch then fails loudly),
    and the next good capture instantiates afresh."""
    cache, host, dp = _setup()
    dec = DecodeEmulator("cuda:0", weight_bytes=64 << 20)
    bad = torch.zeros(1, dtype=torch.int32, device="cuda:0")
    g = DecodeGraph("cuda:0", marks=2 * GEO.num_planes)
    comp = torch.cuda.Stream()
    good = np.array([[3, 0, 40, 5]], dtype=np.int64)
    dp.kv_tokens(0, good, stream=comp)
    comp.synchronize()
    assert g.capture_step(dp, dec, good, bad.data_ptr(), 1 << 20) == 2
    g.launch(comp)
    comp.synchronize()
    with pytest.raises(IndexError):
        g.capture_step(dp, dec, np.array([[3, 0, 40, 63]], dtype=np.int64), bad.data_ptr(),
                       1 << 20)
    with pytest.raises(ValueError):
        g.launch(comp)
    assert g.capture_step(dp, dec, good, bad.data_ptr(), 1 << 20) == 2
    g.launch(comp)
    comp.synchronize()
    assert int(bad.item()) == 0
    g.close()
    host.close()
