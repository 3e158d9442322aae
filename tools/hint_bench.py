"""Host-access variant experiment: per-direction GB/s of the LSU swap kernel
for the KVS_HINT_OUT / KVS_HINT_IN variants (set in the environment).

python tools/hint_bench.py --blocks 2048   -> one JSON line
"""

import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import bytes_oracle as orc  # noqa: E402  (plan generator + checker)
from paper_2411_18424_b200.dataplane import HostKVPool, PagedKVCache, SwapDataPlane  # noqa: E402
from paper_2411_18424_b200.geometry import PRESETS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--blocks", type=int, default=2048)
    ap.add_argument("--group", type=int, default=16)
    ap.add_argument("--ctas", default="8,32,148")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    geo = PRESETS["llama3-8b"]
    pool = 2 * args.blocks
    cache = PagedKVCache(geo, pool, device="cuda:0")
    host = HostKVPool(pool, geo.block_bytes)
    dp = SwapDataPlane(cache, host)
    cache.planes.view(torch.int32).random_()
    rng = np.random.default_rng(3)
    ops = orc.random_runs(rng, args.blocks, args.group, pool, pool).astype(np.int32)
    s = torch.cuda.Stream()
    nbytes = args.blocks * geo.block_bytes
    res = {"hint_out": os.environ.get("KVS_HINT_OUT", "0"),
           "hint_in": os.environ.get("KVS_HINT_IN", "0")}
    for ctas in [int(c) for c in args.ctas.split(",")]:
        for d in ("out", "in"):
            dp.set_launch(d, ctas, 512)
            dp.swap(d, ops, stream=s)
            s.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(args.reps):
                dp.swap(d, ops, stream=s)
            e1.record(s)
            s.synchronize()
            res[f"{d}_{ctas}"] = round(nbytes * args.reps / (e0.elapsed_time(e1) * 1e-3) / 1e9, 2)
    # bytes check of the last round trip
    snap = cache.planes.clone()
    dp.swap("out", ops, stream=s)
    cache.planes.fill_(0)
    dp.swap("in", ops, stream=s)
    s.synchronize()
    rows = np.concatenate([np.arange(g, g + b) for b, g, c in ops])
    res["roundtrip_exact"] = bool(torch.equal(snap[:, rows], cache.planes[:, rows]))
    print(json.dumps(res), flush=True)
    dp.close()
    host.close()


if __name__ == "__main__":
    main()
