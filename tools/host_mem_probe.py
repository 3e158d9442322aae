"""Host pool flavour vs PCIe throughput: cudaHostAlloc (default), cudaHostAlloc
WriteCombined (not snooped), mmap + cudaHostRegister.  Kernel per direction,
kernel duplex, copy engines, and an exact round trip per flavour.

python tools/host_mem_probe.py --blocks 2048   -> JSON lines
"""

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_18424_b200 import synthetic as orc  # noqa: E402  (plan generator)
from paper_2411_18424_b200.dataplane import HostKVPool, PagedKVCache, SwapDataPlane  # noqa: E402
from paper_2411_18424_b200.geometry import PRESETS  # noqa: E402


def timed(streams_fns, reps=3):
    evs = []
    for s, fn in streams_fns:
        fn()
    torch.cuda.synchronize()
    for s, fn in streams_fns:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            fn()
        e1.record(s)
        evs.append((e0, e1))
    torch.cuda.synchronize()
    return [e0.elapsed_time(e1) / reps * 1e-3 for e0, e1 in evs]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--blocks", type=int, default=2048)
    args = ap.parse_args()
    geo = PRESETS["llama3-8b"]
    n = args.blocks
    cache = PagedKVCache(geo, 2 * n, device="cuda:0")
    cache.planes.view(torch.int32).random_()
    torch.cuda.synchronize()
    rng = np.random.default_rng(4)
    ops = orc.random_runs(rng, n, 16, 2 * n, 2 * n).astype(np.int32)
    half = n // 2
    ops_a = orc.random_runs(rng, half, 16, n, n).astype(np.int32)
    ops_b = ops_a.copy()
    ops_b[:, 1:] += n
    nbytes = n * geo.block_bytes
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for flavour in ("default", "write_combined", "register"):
        host = HostKVPool(2 * n, geo.block_bytes, write_combined=flavour == "write_combined",
                          register=flavour == "register")
        dp = SwapDataPlane(cache, host)
        row = {"host": flavour}
        for name, (co, ci) in {"8x512|8x256": ((8, 512), (8, 256)),
                               "32x512": ((32, 512), (32, 512))}.items():
            dp.set_launch("out", *co)
            dp.set_launch("in", *ci)
            t_out, = timed([(s1, lambda: dp.swap("out", ops, stream=s1))])
            t_in, = timed([(s1, lambda: dp.swap("in", ops, stream=s1))])
            row[f"out_{name}"] = round(nbytes / t_out / 1e9, 2)
            row[f"in_{name}"] = round(nbytes / t_in / 1e9, 2)
        dp.set_launch("out", 32, 512)
        dp.set_launch("in", 32, 512)
        hb = half * geo.block_bytes
        t_o, t_i = timed([(s1, lambda: dp.swap("out", ops_a, stream=s1)),
                          (s2, lambda: dp.swap("in", ops_b, stream=s2))])
        row["duplex_kernel"] = {"out": round(hb / t_o / 1e9, 2), "in": round(hb / t_i / 1e9, 2)}
        t_out, = timed([(s1, lambda: dp.baseline("out", 1, ops, stream=s1))])
        t_in, = timed([(s1, lambda: dp.baseline("in", 1, ops, stream=s1))])
        row["ce_per_run"] = {"out": round(nbytes / t_out / 1e9, 2), "in": round(nbytes / t_in / 1e9, 2)}
        t_o, t_i = timed([(s1, lambda: dp.baseline("out", 2, ops_a, stream=s1)),
                          (s2, lambda: dp.baseline("in", 2, ops_b, stream=s2))])
        row["duplex_ce_staged"] = {"out": round(hb / t_o / 1e9, 2), "in": round(hb / t_i / 1e9, 2)}
        # exact round trip through this pool (checked on the GPU: no CPU reads of WC memory)
        dp.set_launch("out", 0, 0)
        dp.set_launch("in", 0, 0)
        rows = torch.from_numpy(np.concatenate([np.arange(g, g + b) for b, g, c in ops])).cuda()
        snap = cache.planes[:, rows].clone()
        dp.swap("out", ops, stream=s1)
        s1.synchronize()
        cache.planes[:, rows] = 0
        torch.cuda.synchronize()
        dp.swap("in", ops, stream=s1)
        s1.synchronize()
        row["roundtrip_exact"] = bool(torch.equal(snap, cache.planes[:, rows]))
        print(json.dumps(row), flush=True)
        dp.close()
        host.close()


if __name__ == "__main__":
    main()
