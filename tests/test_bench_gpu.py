"""bench.py's N>1 path on one GPU: two ranks under torchrun (gloo for the
plumbing, both on cuda:0) run the kernel steps, the e2e leg and the TP
lockstep trace; rank 0 prints one JSON line.  A code-path check — two ranks
sharing one GPU and one PCIe link say nothing about scaling."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def test_bench_two_ranks_one_line(cuda_ok):
    """`bench.py --gpus 2` with no launcher relaunches itself as two ranks."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["KVS_BENCH_BACKEND"] = "gloo"
    cmd = [sys.executable, "bench.py", "--gpus", "2", "--steps", "1", "--warmup", "3",
           "--plan-blocks", "1024", "--no-sweep", "--no-cpu-baseline", "--trace-convs", "6",
           "--traces", "stress_vtc"]
    res = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["scaling"] == "weak"
    assert d["backend"] == "gloo"
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] > 0 and d["e2e"]["bytes_verified"]
    assert d["e2e_serving"]["bytes_verified"]
    assert len(d["roofline"]["aggregate"]["ce_per_rank_gbs"]) == 2
    tr = d["trace"]["stress_vtc"]
    assert tr["tp"] == 2 and tr["pattern"] == "vtc"
    for run in tr["runs"].values():
        assert run["tokens"] > 0 and run["ttft_p99_ms"] > 0
