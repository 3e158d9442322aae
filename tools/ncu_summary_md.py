"""Render profiles/ncu_kernel_summary.json as the top section of
profiles/r01_ncu_summary.md (keeps the TMA-bulk section below it).

python tools/ncu_summary_md.py <raw-csv-name> <launch-list-name>
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
raw, launches = sys.argv[1], sys.argv[2]
d = json.load(open(ROOT / "profiles" / "ncu_kernel_summary.json"))
md = ROOT / "profiles" / "r01_ncu_summary.md"
_, sep, rest = md.read_text().partition("## TMA bulk kernel")
ko, ki = d["kernels"]["out"], d["kernels"]["in"]
lines = ["# ncu --set full: swap kernels (round 1, final kernel code)", "",
         f"Source: `{d['source']}` (`ncu --set full --clock-control none --import-source on "
         "-k regex:kvs_swap_kernel -c 2`, `bench.py --steps 1 --warmup 0 --no-sweep "
         "--no-cpu-baseline --no-trace --sm-partition 0`): one 4096-block (8 GiB) plan each way, "
         f"LLaMA-3-8B KV (2 MiB blocks), runs of 16. Raw page: `{raw}`; launch list: `{launches}`.",
         "", "| metric | swap-out `kvs_swap_kernel<0>` | swap-in `kvs_swap_kernel<1>` |",
         "|---|---:|---:|"]
for k in sorted(set(ko["raw"]) | set(ki["raw"])):
    a, b = ko["raw"].get(k, {}), ki["raw"].get(k, {})
    lines.append(f"| `{k}` | {a.get('value', '')} {a.get('unit', '')} | "
                 f"{b.get('value', '')} {b.get('unit', '')} |")
lines += ["", "Reading:", "",
          f"* payload 8.590 GB per launch; DRAM traffic {ko['dram_bytes_per_launch'] / 1e9:.3f} "
          f"(out) / {ki['dram_bytes_per_launch'] / 1e9:.3f} GB (in): no re-reads;",
          f"* PCIe wire rate {ko['pcie_write_gbs']:.1f} GB/s (out, writes) / "
          f"{ki['pcie_read_gbs']:.1f} GB/s (in, read completions) for {ko['dram_gbs']:.1f} / "
          f"{ki['dram_gbs']:.1f} GB/s of payload: 128 B TLPs, the SM-path ceiling (~53 GB/s of "
          "payload on a 63 GB/s link);",
          f"* the swap-in's upstream direction carries {ki['pcie_write_gbs']:.1f} GB/s of read "
          "requests (one per 128 B);",
          "* SM throughput is a fraction of a percent: the kernels are link-bound, not issue-bound.",
          "", ""]
md.write_text("\n".join(lines) + sep + rest)
