"""Hottest SASS instructions of one kernel from an ncu report (source page),
with their dominant stall reasons and shared-memory wavefronts vs ideal.
Usage: python tools/ncu_sass_hot.py rep.ncu-rep kernel-regex [top] [samples|exec]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source",
                      "sass", "-k", "regex:" + sys.argv[2]], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
col = {k: i for i, k in enumerate(h)}
ia, isrc, iex, ismp = (col["Address"], col["Source"], col["Instructions Executed"],
                       col["Warp Stall Sampling (All Samples)"])
stall_cols = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
data = [r for r in rows[2:] if len(r) > iex and r[iex].isdigit()]


def num(r, k):
    try:
        return float(r[col[k]].replace(",", "") or 0)
    except (KeyError, ValueError):
        return 0.0


tot = sum(int(r[iex]) for r in data)
stot = sum(int(r[ismp] or 0) for r in data)
wf = sum(num(r, "L1 Wavefronts Shared") for r in data)
wfi = sum(num(r, "L1 Wavefronts Shared Ideal") for r in data)
print(f"total warp instructions {tot}, samples {stot}, shared wavefronts {wf:.0f} (ideal {wfi:.0f})")
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
key = (lambda r: -int(r[ismp] or 0)) if (len(sys.argv) <= 4 or sys.argv[4] == "samples") else (
    lambda r: -int(r[iex]))
for r in sorted(data, key=key)[:top]:
    st = sorted(((num(r, k), k[6:]) for k in stall_cols), reverse=True)[:2]
    sts = " ".join(f"{k}:{v:.0f}" for v, k in st if v > 0)
    w = num(r, "L1 Wavefronts Shared")
    wi = num(r, "L1 Wavefronts Shared Ideal")
    ws = f" smem_wf {w / max(wi, 1):.2f}x" if wi else ""
    print(f"{r[ia][-5:]} {int(r[iex]):>10} {int(r[ismp] or 0):>6}  {r[isrc].strip()[:60]:<60} {sts}{ws}")
