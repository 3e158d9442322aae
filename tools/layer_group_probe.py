"""Swap GB/s of plane-major (layered) order vs plane-group size, against
block-major kvs_swap: strict plane-major reads 64 KiB of host memory every
2 MiB (LLaMA-3-8B blocks); groups of g planes read g x 64 KiB runs."""

import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_18424_b200 import synthetic as orc  # noqa: E402  (plan generator)
from paper_2411_18424_b200.dataplane import HostKVPool, PagedKVCache, SwapDataPlane  # noqa: E402
from paper_2411_18424_b200.geometry import PRESETS  # noqa: E402


def main():
    geo = PRESETS[sys.argv[1] if len(sys.argv) > 1 else "llama3-8b"]
    n = 2048
    cache = PagedKVCache(geo, 2 * n, device="cuda:0")
    host = HostKVPool(2 * n, geo.block_bytes)
    dp = SwapDataPlane(cache, host)
    dp.set_launch("out", 8, 512)
    dp.set_launch("in", 8, 256)
    flags = torch.zeros(geo.num_planes, dtype=torch.int32, device="cuda:0")
    rng = np.random.default_rng(6)
    ops = orc.random_runs(rng, n, 16, 2 * n, 2 * n).astype(np.int32)
    s = torch.cuda.Stream()
    nbytes = n * geo.block_bytes
    seq = [0]

    def rate(fn):
        fn()
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(3):
            fn()
        e1.record(s)
        s.synchronize()
        return round(3 * nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9, 2)

    def layered(d):
        seq[0] += 1
        dp.swap_layered(d, ops, flags.data_ptr(), seq[0], stream=s)

    row = {"model": geo.name, "chunk": geo.plane_chunk_bytes}
    for d in ("out", "in"):
        row[f"{d}_block_major"] = rate(lambda: dp.swap(d, ops, stream=s))
        for g in (1, 2, 4, 8, 0):
            dp.set_layer_group(g)
            row[f"{d}_layered_g{g or 'auto'}"] = rate(lambda: layered(d))
    dp.set_layer_group(0)
    print(json.dumps(row), flush=True)
    host.close()


if __name__ == "__main__":
    main()
