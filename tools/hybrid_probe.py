"""Single-direction hybrid: split one plan's runs between the LSU kernel and
the copy engines (one cudaMemcpy2DAsync per (plane, run)), concurrently on two
streams.  SM-issued host traffic leaves in 128 B TLPs (~53 GB/s payload
ceiling), the copy engines in 256 B ones (~57): does a mix carry more than
either alone?"""

import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_18424_b200 import synthetic as orc  # noqa: E402  (plan generator)
from paper_2411_18424_b200.dataplane import HostKVPool, PagedKVCache, SwapDataPlane  # noqa: E402
from paper_2411_18424_b200.geometry import LLAMA3_8B  # noqa: E402


def main():
    geo = LLAMA3_8B
    n = 2048
    cache = PagedKVCache(geo, 2 * n, device="cuda:0")
    host = HostKVPool(2 * n, geo.block_bytes)
    dp = SwapDataPlane(cache, host)
    rng = np.random.default_rng(8)
    ops = orc.random_runs(rng, n, 64, 2 * n, 2 * n).astype(np.int32)  # 32 runs of 64 blocks
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    nbytes = n * geo.block_bytes
    for d in ("out", "in"):
        dp.set_launch(d, 32, 512)
        for frac_ce in (0.0, 0.25, 0.4, 0.5, 0.6, 0.75, 1.0):
            k = int(round(len(ops) * frac_ce))
            ce_ops, k_ops = ops[:k], ops[k:]

            def go():
                if len(k_ops):
                    dp.swap(d, k_ops, stream=s1)
                if len(ce_ops):
                    dp.baseline(d, 1, ce_ops, stream=s2)
            go()
            torch.cuda.synchronize()
            ref = torch.cuda.Event(enable_timing=True)
            ref.record()
            torch.cuda.synchronize()
            ends = []
            for _ in range(3):
                go()
            e1, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e1.record(s1)
            e2.record(s2)
            torch.cuda.synchronize()
            span = max(ref.elapsed_time(e1), ref.elapsed_time(e2)) * 1e-3
            print(json.dumps({"dir": d, "ce_fraction": frac_ce,
                              "gbs": round(3 * nbytes / span / 1e9, 2)}), flush=True)
    host.close()


if __name__ == "__main__":
    main()
