"""Per-plan latency of the swap path: one plan of B blocks, end to end on its
stream (launch + op-counter memset + kernel + flag publication), for the
executor's kvs_swap_ops path, plain kvs_swap and the staged copy-engine path.
Small plans (TP8 shards, short contexts) are latency-, not bandwidth-bound.

python tools/latency_probe.py --model llama3-70b --tp 8   -> one JSON line
"""

import argparse
import json
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_18424_b200 import synthetic as orc  # noqa: E402  (plan generator)
from paper_2411_18424_b200.dataplane import HostKVPool, PagedKVCache, SwapDataPlane  # noqa: E402
from paper_2411_18424_b200.geometry import PRESETS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama3-70b")
    ap.add_argument("--tp", type=int, default=8)
    ap.add_argument("--blocks", default="1,4,16,64,256")
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    geo = PRESETS[args.model].with_tp(args.tp)
    pool = 2048
    cache = PagedKVCache(geo, pool, device="cuda:0")
    host = HostKVPool(pool, geo.block_bytes)
    dp = SwapDataPlane(cache, host)
    flags = torch.zeros(4096, dtype=torch.int32, device="cuda:0")
    s = torch.cuda.Stream()
    rng = np.random.default_rng(0)
    res = {"model": geo.name, "tp": args.tp, "block_bytes": geo.block_bytes, "rows": []}
    for b in [int(x) for x in args.blocks.split(",")]:
        ops = orc.random_runs(rng, b, max(1, b // 4), pool, pool).astype(np.int32)
        row = {"blocks": b, "mib": round(b * geo.block_bytes / 2**20, 2), "ops": len(ops)}
        for d in ("out", "in"):
            impls = {
                "kernel_ops": lambda: dp.swap_ops(d, ops, flags.data_ptr(), 1, stream=s),
                "kernel": lambda: dp.swap(d, ops, stream=s),
                "ce_staged": lambda: dp.baseline(d, 2, ops, stream=s),
            }
            for name, fn in impls.items():
                fn()
                s.synchronize()
                ts = []
                for _ in range(args.reps):
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(s)
                    fn()
                    e1.record(s)
                    s.synchronize()
                    ts.append(e0.elapsed_time(e1) * 1e3)
                row[f"{d}_{name}_us"] = round(statistics.median(ts), 1)
        print(json.dumps(row), flush=True)
        res["rows"].append(row)
    host.close()


if __name__ == "__main__":
    main()
