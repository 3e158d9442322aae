"""Layer-wise pipelined swap-in vs iteration-wise swap-in.

A resumed request's KV (B blocks, LLaMA-3-8B shape) is swapped in while its
first decode step runs layer by layer.  Each "layer" of decode streams that
layer's weight slice (weights/num_layers) plus the request's KV of the
layer, then the next layer starts.

  serial   : kvs_swap (whole plan) -> event -> 32 layer kernels
  layered  : kvs_swap_layered; layer l's kernel waits on plane_flags[l]

Reported: time from swap start to the end of the decode step, both ways.
python tools/layered_bench.py [--blocks 64,256,1024]
"""

import argparse
import ctypes
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_18424_b200 import synthetic as orc  # noqa: E402  (plan generator)
from paper_2411_18424_b200 import _lib  # noqa: E402
from paper_2411_18424_b200.dataplane import HostKVPool, PagedKVCache, SwapDataPlane  # noqa: E402
from paper_2411_18424_b200.geometry import PRESETS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--blocks", default="64,256,1024")
    ap.add_argument("--weights-gib", type=int, default=16)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    geo = PRESETS[args.model]
    lib = _lib.load()
    pool = 2048
    cache = PagedKVCache(geo, pool, device="cuda:0")
    host = HostKVPool(pool, geo.block_bytes)
    dp = SwapDataPlane(cache, host)
    cache.planes.view(torch.int32).random_()
    host.array[:] = 1
    weights = torch.empty(args.weights_gib << 30, dtype=torch.uint8, device="cuda:0")
    weights.view(torch.int32).random_()
    sink = torch.zeros(4, dtype=torch.int32, device="cuda:0")
    L = geo.num_planes
    w_layer = weights.numel() // L
    flags = torch.zeros(L, dtype=torch.int32, device="cuda:0")
    s_swap, s_dec = torch.cuda.Stream(), torch.cuda.Stream(priority=-1)
    rng = np.random.default_rng(0)
    seq = 0
    out = []

    def layer_kernel(l, kv_bytes):
        base = weights.data_ptr() + l * w_layer
        rc = lib.kvs_stream_read(0, int(s_dec.cuda_stream), ctypes.c_void_p(base), w_layer,
                                 w_layer + kv_bytes, 0, ctypes.c_void_p(sink.data_ptr()))
        _lib.check(rc)

    for B in [int(x) for x in args.blocks.split(",")]:
        ops = orc.random_runs(rng, B, 16, pool, pool).astype(np.int32)
        kv_layer = B * geo.plane_chunk_bytes
        res = {"blocks": B, "swap_mib": B * geo.block_bytes >> 20}
        for mode in ("serial", "layered", "decode_only", "swap_only"):
            times = []
            for r in range(args.reps + 1):
                seq += 1
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s_swap)
                s_dec.wait_event(e0)
                if mode == "serial":
                    dp.swap("in", ops, stream=s_swap)
                    done = torch.cuda.Event()
                    done.record(s_swap)
                    s_dec.wait_event(done)
                    for l in range(L):
                        layer_kernel(l, kv_layer)
                elif mode == "layered":
                    dp.swap_layered("in", ops, flags.data_ptr(), seq, stream=s_swap)
                    for l in range(L):
                        dp.wait_flag(s_dec, flags.data_ptr() + 4 * l, seq)
                        layer_kernel(l, kv_layer)
                elif mode == "decode_only":
                    for l in range(L):
                        layer_kernel(l, kv_layer)
                else:
                    dp.swap("in", ops, stream=s_swap)
                    done = torch.cuda.Event()
                    done.record(s_swap)
                    s_dec.wait_event(done)
                e1.record(s_dec)
                torch.cuda.synchronize()
                if r:
                    times.append(e0.elapsed_time(e1))
            res[f"{mode}_ms"] = round(float(np.median(times)), 3)
        res["saved_ms"] = round(res["serial_ms"] - res["layered_ms"], 3)
        res["layered_vs_ideal"] = round(res["layered_ms"] / max(res["swap_only_ms"],
                                                                 res["decode_only_ms"]), 3)
        out.append(res)
        print(json.dumps(res), flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/layered_bench.json", "w") as f:
        json.dump(out, f, indent=1)
    host.close()


if __name__ == "__main__":
    main()
