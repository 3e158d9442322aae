"""BASELINE.json configs 3-5 on one B200 (one TP rank's shard; every rank runs
the identical plan stream over its own PCIe link).

  c3  fairness-aware preemption trace (VTC priorities, plus Markov for
      contrast), LLaMA-3-8B KV, async swap overlapped with decode — live mode
  c4  Qwen-2.5-32B KV, TP=2/4/8 per-rank shards, multi-turn reuse
      (dirty-block-only swap-out) — replay mode with real bytes + byte check
  c5  LLaMA-3-70B KV at 32K context, TP8 rank shard, high preemption — live

python tools/config_runs.py c3 c4 c5   -> gpurun_out/config_runs.json
(SM_PARTITION=8 by default: live runs put the swap kernels on their own 8-SM
green context and decode on the rest; SM_PARTITION=0 shares all SMs.
LAYERED=1 by default: FastSwitch runs with layered admission.)
"""

import dataclasses
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2411_18424_b200 import config as mconfig  # noqa: E402
from paper_2411_18424_b200 import engine as engine_mod  # noqa: E402
from paper_2411_18424_b200.engine import Engine  # noqa: E402
from paper_2411_18424_b200.geometry import LLAMA3_8B, LLAMA3_70B, QWEN25_32B  # noqa: E402
from paper_2411_18424_b200.live import DecodeEmulator, LiveEngine, b200_transfer_params  # noqa: E402
from paper_2411_18424_b200.runtime import Runtime  # noqa: E402
from paper_2411_18424_b200.workload import generate  # noqa: E402


SM_PARTITION = int(os.environ.get("SM_PARTITION", "8"))
LAYERED = os.environ.get("LAYERED", "1") == "1"  # FastSwitch runs with layered admission
POLICY = os.environ.get("POLICY", "serving")  # FastSwitch's swap policy (swap.DUPLEX_POLICIES)


def swap_rates(rt):
    ex = rt.executor
    out = {}
    for d in ("out", "in"):
        recs = [r for r in ex.history if r.direction == d and r.nbytes and r.start_event]
        secs = sum(r.start_event.elapsed_time(r.event) for r in recs) * 1e-3
        nb = sum(r.nbytes + r.refresh_bytes for r in recs)
        out[d] = {"gib": round(nb / 2**30, 2), "gbs_while_busy": round(nb / secs / 1e9, 2)
                  if secs else None, "transfers": len(recs)}
    return out


def live_run(geo, doc, impl="kernel", decode=None, verify=False):
    cfg, wl, _ = mconfig.build(doc)
    cfg = dataclasses.replace(cfg, transfer=b200_transfer_params())
    layered = LAYERED and impl == "kernel"
    rt = Runtime(geo, cfg.gpu_pool.total_blocks, cfg.cpu_pool_blocks, copy_impl=impl,
                 verify=verify, timing=True, sm_partition=SM_PARTITION, layered_swap_in=layered,
                 duplex_policy=POLICY if impl == "kernel" else "latency")
    eng = LiveEngine(cfg, generate(wl), rt, decode, layered=layered)
    eng.turn_trace = []
    t0 = time.perf_counter()
    rep = eng.run()
    res = {"wall_s": round(time.perf_counter() - t0, 1), "latency": eng.latency_summary(),
           "ttft_anatomy": eng.ttft_anatomy(),
           "swap": swap_rates(rt), "runtime": rt.stats(),
           "report": {k: rep.to_dict()[k] for k in (
               "total_tokens", "expected_tokens", "swap_out_blocks", "swap_in_blocks",
               "reused_blocks", "avg_granularity_blocks", "conflicts", "sync_stalls")}}
    rt.close()
    return res


def c3(decode):
    base = {"block": {"bytes_per_block": LLAMA3_8B.block_bytes},
            "gpu_pool": {"total_blocks": 512}, "cpu_pool": {"total_blocks": 8192},
            "workload": {"num_conversations": 80, "arrival_rate_per_s": 2.0}}
    out = {}
    for pattern in ("vtc", "markov"):
        doc = {**base, "trace": {"pattern": pattern, "frequency": 0.04}}
        out[pattern] = {"fastswitch": live_run(LLAMA3_8B, {**doc, "ablation": "full"},
                                               decode=decode),
                        "vllm_like": live_run(LLAMA3_8B, {**doc, "ablation": "baseline"},
                                              impl="ce_per_block", decode=decode)}
        print("c3", pattern, json.dumps({k: {m: v["latency"][m] for m in (
            "ttft_p50_ms", "ttft_p99_ms", "tbt_p99_ms", "tbt_p999_ms",
            "swap_induced_decode_stall")} for k, v in out[pattern].items()}), flush=True)
    return out


def c4():
    """Replay with real bytes.  The decisions are first pinned: the report of
    the byte-moving run must equal the golden recorded from the reference
    (tests/golden/engine.json c4_qwen32b_tp*)."""
    golden = json.loads((Path(__file__).resolve().parents[1] / "tests" / "golden"
                         / "engine.json").read_text())
    out = {}
    for tp in (2, 4, 8):
        geo = QWEN25_32B.with_tp(tp)
        want = golden[f"c4_qwen32b_tp{tp}"]
        doc = want["doc"]
        assert doc["block"]["bytes_per_block"] == geo.block_bytes
        cfg, wl, _ = mconfig.build(doc)
        rt = Runtime(geo, cfg.gpu_pool.total_blocks, cfg.cpu_pool_blocks, verify=True,
                     timing=True)
        eng = Engine(cfg, generate(wl), runtime=rt)
        t0 = time.perf_counter()
        rep = eng.run()
        rt.synchronize()
        if json.loads(rep.to_json()) != want["report"]:
            raise AssertionError(f"c4 tp{tp}: replay report differs from the reference golden")
        out[f"tp{tp}"] = {
            "decisions_match_reference_golden": True,
            "block_bytes_per_rank": geo.block_bytes, "heads_per_rank": geo.heads_per_rank,
            "wall_s": round(time.perf_counter() - t0, 1),
            "moved_out_blocks": rep.swap_out_blocks, "reused_blocks": rep.reused_blocks,
            "refresh_blocks": eng.store.refreshed_blocks, "swap_in_blocks": rep.swap_in_blocks,
            "verified_swap_ins": rt.verified, "swap": swap_rates(rt),
            "sim_ttft_p99_ms": rep.ttft_p99_us / 1e3}
        print("c4", tp, json.dumps(out[f"tp{tp}"]), flush=True)
        rt.close()
    return out


def c5(decode):
    geo = LLAMA3_70B.with_tp(8)
    doc = {"ablation": "full", "block": {"bytes_per_block": geo.block_bytes},
           "gpu_pool": {"total_blocks": 8192, "initial_group_blocks": 60},
           "cpu_pool": {"total_blocks": 65536},
           "workload": {"num_conversations": 24, "arrival_rate_per_s": 1.0,
                        "input_tokens": {"median": 6000.0, "sigma": 0.9, "max": 16384},
                        "max_context_tokens": 32768},
           "trace": {"pattern": "random", "frequency": 0.04}}
    res = live_run(geo, doc, decode=decode)
    res["block_bytes_per_rank"] = geo.block_bytes
    print("c5", json.dumps({k: res[k] for k in ("latency", "swap")}), flush=True)
    return res


def main():
    which = sys.argv[1:] or ["c3", "c4", "c5"]
    out = {}
    decode = None
    if "c3" in which or "c5" in which:
        stream, ctas = None, 0
        if SM_PARTITION:
            from paper_2411_18424_b200.swap import partition_streams
            _, stream, sms = partition_streams(torch.device("cuda:0"), SM_PARTITION)
            ctas = 2 * sms[1]
            out["sm_partition"] = sms
        decode = DecodeEmulator("cuda:0", weight_bytes=16 << 30, ctas=ctas, stream=stream)
        out["decode_calibrated_gbs"] = round(decode.bytes_per_us / 1e3, 1)
    if "c4" in which:
        out["c4"] = c4()
    if "c3" in which:
        out["c3"] = c3(decode)
    if "c5" in which:
        out["c5"] = c5(decode)
    os.makedirs("gpurun_out", exist_ok=True)
    path = "gpurun_out/config_runs.json"
    with open(path, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
