"""Full-duplex mixes: which engine per direction reaches the most combined
host-link GB/s when a swap-out and a swap-in run at once (LSU kernel, TMA
bulk kernel, copy-engine staged path)."""

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
    geo = PRESETS["llama3-8b"]
    n = 2048
    cache = PagedKVCache(geo, 2 * n, device="cuda:0")
    host = HostKVPool(2 * n, geo.block_bytes)
    dp = SwapDataPlane(cache, host)
    rng = np.random.default_rng(4)
    ops_a = orc.random_runs(rng, n, 16, n, n).astype(np.int32)
    ops_b = ops_a.copy()
    ops_b[:, 1:] += n
    hb = n * geo.block_bytes
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    engines = {
        "lsu": lambda d, ops, s: dp.swap(d, ops, stream=s),
        "bulk": lambda d, ops, s: dp.swap(d, ops, stream=s),
        "ce": lambda d, ops, s: dp.baseline(d, 2, ops, stream=s),
    }
    for eo, ei in (("lsu", "lsu"), ("lsu", "ce"), ("ce", "lsu"), ("lsu", "bulk"), ("bulk", "lsu"),
                   ("bulk", "bulk"), ("ce", "ce")):
        for d, e in (("out", eo), ("in", ei)):
            dp.set_path(d, "bulk" if e == "bulk" else "lsu")
            dp.set_launch(d, 32 if e == "lsu" else 64, 512 if e == "lsu" else 0)
        fo = lambda: engines[eo]("out", ops_a, s1)
        fi = lambda: engines[ei]("in", ops_b, s2)
        fo(); fi()
        torch.cuda.synchronize()
        ref = torch.cuda.Event(enable_timing=True)
        ref.record()
        torch.cuda.synchronize()
        ev = {k: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for k in ("out", "in")}
        ev["out"][0].record(s1); ev["in"][0].record(s2)
        for _ in range(3):
            fo(); fi()
        ev["out"][1].record(s1); ev["in"][1].record(s2)
        torch.cuda.synchronize()
        t = {k: ev[k][0].elapsed_time(ev[k][1]) * 1e-3 for k in ev}
        span = (max(ref.elapsed_time(ev[k][1]) for k in ev) -
                min(ref.elapsed_time(ev[k][0]) for k in ev)) * 1e-3
        row = {"out": eo, "in": ei,
               "out_gbs": round(3 * hb / t["out"] / 1e9, 2), "in_gbs": round(3 * hb / t["in"] / 1e9, 2),
               "combined_gbs_union": round(6 * hb / span / 1e9, 2)}
        print(json.dumps(row), flush=True)
    host.close()


if __name__ == "__main__":
    main()
