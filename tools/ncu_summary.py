"""Summarise an ncu --set full capture of the kvs_swap kernels into
profiles/ncu_kernel_summary.json (+ a markdown table on stdout).

python tools/ncu_summary.py gpurun_out/prof.ncu-rep [output name under profiles/]
"""

import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

WANT = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "pcie__read_bytes.sum.per_second",
    "pcie__write_bytes.sum.per_second",
    "dram__bytes.sum.per_second",
    "lts__t_sectors_aperture_sysmem.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__grid_size",
    "launch__block_size",
    "launch__registers_per_thread",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard",
]


def raw_rows(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    header, units = rows[0], rows[1]
    return header, units, rows[2:]


def to_num(s: str):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return s


def main():
    rep = sys.argv[1]
    header, units, rows = raw_rows(rep)
    idx = {h: i for i, h in enumerate(header)}
    kernels = {}
    for r in rows:
        name = r[idx["Kernel Name"]]
        if "kvs_swap_kernel" not in name:
            continue
        direction = "out" if "kvs_swap_kernelILi0" in name or "<0," in name else "in"
        m = {}
        for key in WANT:
            if key in idx:
                m[key] = {"value": to_num(r[idx[key]]), "unit": units[idx[key]]}
        kernels.setdefault(direction, []).append(m)
    summary = {"source": rep, "kernels": {}}
    for d, lst in kernels.items():
        m = lst[0]

        def val(k, scale=1.0):
            v = m.get(k, {}).get("value")
            u = m.get(k, {}).get("unit", "")
            if not isinstance(v, float):
                return None
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9,
                    "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "usecond": 1e-6,
                    "msecond": 1e-3, "second": 1.0, "byte/s": 1.0, "Kbyte/s": 1e3,
                    "Mbyte/s": 1e6, "Gbyte/s": 1e9}.get(u, 1.0)
            return v * mult * scale
        dram = (val("dram__bytes_read.sum") or 0) + (val("dram__bytes_write.sum") or 0)
        summary["kernels"][d] = {
            "launches_profiled": len(lst),
            "duration_s": val("gpu__time_duration.sum"),
            "dram_bytes_per_launch": dram,
            "dram_read_bytes": val("dram__bytes_read.sum"),
            "dram_write_bytes": val("dram__bytes_write.sum"),
            "pcie_read_gbs": (val("pcie__read_bytes.sum.per_second") or 0) / 1e9,
            "pcie_write_gbs": (val("pcie__write_bytes.sum.per_second") or 0) / 1e9,
            "dram_gbs": (val("dram__bytes.sum.per_second") or 0) / 1e9,
            "raw": m,
        }
    out = ROOT / "profiles" / (sys.argv[2] if len(sys.argv) > 2 else "ncu_kernel_summary.json")
    out.parent.mkdir(exist_ok=True)
    out.write_text(json.dumps(summary, indent=1))
    for d, k in summary["kernels"].items():
        print(d, {kk: vv for kk, vv in k.items() if kk != "raw"})


if __name__ == "__main__":
    main()
