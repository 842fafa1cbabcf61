"""Print selected raw ncu metrics (regex on the metric name) for each kernel of
a report.  Usage: python tools/ncu_grep.py rep.ncu-rep 'regex' [kernel-regex]"""
import csv
import io
import re
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
pat = re.compile(sys.argv[2])
kpat = re.compile(sys.argv[3]) if len(sys.argv) > 3 else None
seen = set()
for r in rows[2:]:
    name = r[h.index("Kernel Name")]
    if kpat and not kpat.search(name):
        continue
    if name in seen:
        continue
    seen.add(name)
    print(name[:60])
    for i, k in enumerate(h):
        if pat.search(k) and r[i] not in ("", "0", "0.000000"):
            print(f"   {k} = {r[i]} {units[i]}")
