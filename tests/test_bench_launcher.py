"""bench.py's launcher and reference arm on CPU (no GPU needed).

`python bench.py --gpus N` without torchrun must become N ranks itself, rank
0 alone printing one line with n_gpus = N; a launcher that started a
different number of ranks must fail loudly.  The reference arm moves the GPU
arm's own plans (same seed, sizes, pools) with the oracle's C restatement and
times the reference's control plane per call (baseline/_ref when installed)."""

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def _bench(*args, env=None):
    e = {k: v for k, v in os.environ.items()
         if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    e.update(env or {})
    return subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, env=e,
                          capture_output=True, text=True, timeout=600)


def test_gpus_2_without_torchrun_relaunches_two_ranks_one_line():
    res = _bench("--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0",
                 "--plan-blocks", "128")
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    cb = d["cpu_baseline"]
    assert cb["cores"] >= 1 and cb["cpu_count"] == os.cpu_count() and "numa_node" in cb
    cp = cb["control_plane"]
    assert "unavailable" in cp or (cp["plan_swap_out_us"] > 0 and cp["iter_us"] > 0)
    assert d["config"]["plan_blocks"] == 128 and d["e2e"]["h2d_bytes_per_step"] == 0


def test_launcher_rank_count_mismatch_fails_loudly():
    res = _bench("--impl", "reference", "--gpus", "4", "--steps", "1", "--warmup", "0",
                 env={"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert res.returncode != 0
    assert "WORLD_SIZE=2" in res.stderr


def test_reference_arm_plans_are_the_gpu_arms_plans():
    sys.path.insert(0, str(ROOT))
    import bench
    from oracle.bytes_oracle import random_runs, table_to_ops

    for g in (1, 16, 256):
        ours = bench.make_plans(g, 0)
        ref = bench.make_plans(g, 0, runs=random_runs, pair=table_to_ops)
        for a, b in zip(ours, ref):
            assert (a == b).all()


def test_control_plane_cost_times_each_hot_call():
    sys.path.insert(0, str(ROOT))
    import bench

    ours = bench.control_plane_cost("ours")
    for k in ("plan_swap_out", "plan_swap_in", "allocate", "dispatch"):
        assert ours[f"{k}_calls"] > 0 and ours[f"{k}_us"] > 0
    assert ours["iterations"] > 1000 and ours["iter_us"] > 0
    ref = bench.control_plane_cost("reference")
    if "unavailable" not in ref:  # baseline/_ref installed: same trace, same call counts
        for k in ("plan_swap_out", "plan_swap_in", "allocate", "dispatch"):
            assert ref[f"{k}_calls"] == ours[f"{k}_calls"]
        assert ref["iterations"] == ours["iterations"]
