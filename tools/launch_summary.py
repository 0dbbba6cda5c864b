"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel
launch count, mean duration and share of the library's (mhfd::) device time.
Usage: python tools/launch_summary.py launches.csv > profiles/rNN_launches.txt"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr, data = rows[0], rows[1:]
iK, iV, iU = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
agg = collections.defaultdict(list)
for r in data:
    name = r[iK].split("(")[0].replace("void ", "").replace("mhfd::", "")
    if not name.startswith("k_"):
        continue   # synthetic-input generation (torch) is outside the timed step
    agg[name].append(float(r[iV].replace(",", "")) * scale[r[iU]])
tot = sum(sum(v) for v in agg.values())
print(f"# {sys.argv[1]}: library kernels (k_*) only (cold-cache, serialised ncu timings; compare shares)")
print(f"{'kernel':40s} {'launches':>8s} {'mean_ms':>10s} {'share':>7s}")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:40s} {len(v):8d} {sum(v) / len(v):10.4f} {sum(v) / tot * 100:6.1f}%")
