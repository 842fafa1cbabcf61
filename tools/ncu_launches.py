"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list into
per-kernel counts, mean durations and shares.  Usage:
python tools/ncu_launches.py gpurun_out/launches.csv [> profiles/...md]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
    name = name.split("::")[-1]
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
tot = sum(v[1] for v in agg.values())
print("| kernel | launches | mean (us) | total (ms) | share |")
print("|---|---|---|---|---|")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"| {k} | {n} | {t / n:.2f} | {t / 1e3:.3f} | {100 * t / tot:.1f}% |")
print(f"\ntotal kernel time {tot / 1e3:.2f} ms over {sum(v[0] for v in agg.values())} launches")
