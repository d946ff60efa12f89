"""Markdown summary of an ncu launch list (``--metrics gpu__time_duration.sum
--csv``): per kernel, launches, share of the listed GPU time, average and
median duration (measurement aid).

    python tools/launch_summary.py launches.csv "command line" [headline-kernel-substring]
"""
import csv
import statistics
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
times = defaultdict(list)
for r in rows[hdr + 1:]:
    if len(r) > vi:
        v = float(r[vi].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
        name = r[ki].replace("void ", "").split("(")[0]
        times[name].append(v)
tot = sum(sum(v) for v in times.values())
print(f"# Launch list: `ncu --metrics gpu__time_duration.sum --clock-control none` of `{sys.argv[2]}`\n")
if len(sys.argv) > 3:
    hk = [k for k in times if sys.argv[3] in k]
    for k in hk:
        v = times[k]
        big = [t for t in v if t >= 0.5 * max(v)]  # the full-stream launches (the rest: end-to-end chunks)
        print(f"* headline kernel `{k}`: {len(v)} launches; the {len(big)} full-stream ones median "
              f"{statistics.median(big):.1f} us (cold caches, serialised)")
    print()
print("| share | launches | avg us | median us | kernel |\n|---|---|---|---|---|")
for k, v in sorted(times.items(), key=lambda kv: -sum(kv[1])):
    print(f"| {100 * sum(v) / tot:.1f}% | {len(v)} | {sum(v) / len(v):.1f} | {statistics.median(v):.1f} | `{k[:110]}` |")
