"""Executed-instruction mix by opcode (and the hottest address ranges) of one
kernel from an ncu report's SASS source page.
Usage: python tools/ncu_opmix.py rep.ncu-rep kernel-regex [top]"""
import collections
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source",
                      "sass", "-k", "regex:" + sys.argv[2]], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
col = {k: i for i, k in enumerate(h)}
ie, isrc, ia = col["Instructions Executed"], col["Source"], col["Address"]
seen = {}
for r in rows[2:]:
    if len(r) > ie and r[ie].isdigit():
        seen.setdefault(r[ia], r)
data = sorted(seen.values(), key=lambda r: int(r[ia], 16))
tot = sum(int(r[ie]) for r in data)
print("executed warp instructions", tot)
by = collections.Counter()
for r in data:
    w = r[isrc].split()
    op = w[1] if w[0].startswith("@") else w[0]
    by[op.split(".")[0]] += int(r[ie])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
for k, v in by.most_common(top):
    print(f"  {k:12s} {100 * v / tot:5.1f}%")
# blocks of consecutive instructions with equal execution counts (basic blocks)
print("hottest basic blocks (count x length):")
blocks, cur = [], None
for r in data:
    c = int(r[ie])
    if cur and cur[1] == c:
        cur[2] += 1
    else:
        cur = [r[ia], c, 1]
        blocks.append(cur)
for a, c, n in sorted(blocks, key=lambda b: -b[1] * b[2])[:15]:
    print(f"  {a} count {c} len {n} share {100 * c * n / tot:5.1f}%")
