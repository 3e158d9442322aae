"""Summarise an ncu `--metrics gpu__time_duration.sum` launch list (CSV) into
per-kernel totals and shares.  python tools/launch_summary.py launches.csv > out.md"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
gi, bi = h.index("Grid Size"), h.index("Block Size")
tot, cnt, shape = defaultdict(float), defaultdict(int), {}
scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0][:70]
    tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
    cnt[name] += 1
    shape[name] = f"grid {r[gi]} block {r[bi]}"
all_ms = sum(tot.values())
print(f"# ncu launch list: {sys.argv[1]}\n")
print(f"{sum(cnt.values())} launches, {all_ms:.2f} ms total device time "
      "(cold-cache, serialised under ncu: compare shares, not absolutes)\n")
print("| kernel | launches | total ms | mean ms | share | launch shape |")
print("|---|---:|---:|---:|---:|---|")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"| `{k}` | {cnt[k]} | {tot[k]:.2f} | {tot[k] / cnt[k]:.3f} | "
          f"{100 * tot[k] / all_ms:.1f}% | {shape[k]} |")
