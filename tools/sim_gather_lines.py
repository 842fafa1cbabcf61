"""CPU model of the sweep's gather locality: distinct 128-byte lines per
gather instruction for lane mappings P particles x E lanes.
Usage: python tools/sim_gather_lines.py"""
import sys; sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import numpy as np
from scipy.spatial import cKDTree
from paper_1804_07598_b200 import inputs
s = inputs.lj_lattice_system(40, 40, 40, jitter_key=(2,), vel_key=(102,))
rng = np.random.default_rng(0)
x = s.pos[:, :3].astype(np.float64) + rng.normal(0, 0.12, (s.n, 3))
L = (s.hi - s.lo).astype(np.float64)
x = np.mod(x, L)
rv = 2.8
n = np.floor(L / rv).astype(int)
w = L / n
c = np.minimum((x / w).astype(int), n - 1)
cid = c[:, 0] + n[0] * (c[:, 1] + n[1] * c[:, 2])
order = np.lexsort((np.arange(s.n), cid))
x = x[order]
tree = cKDTree(x, boxsize=L)
nb = tree.query_ball_point(x, rv)
rows = [np.array(sorted(j for j in nb[i] if j != i)) for i in range(s.n)]
def cost(P, E, nw=400):
    # warp = P particles x E lanes each; lane (p, r) loads entries r, r+E, ...
    tot = 0; ninst = 0; entries = 0
    starts = rng.choice(s.n // P, nw, replace=False) * P
    for b in starts:
        rs = [rows[b + p] for p in range(P)]
        K = max((len(r) + E - 1) // E for r in rs)
        for k in range(K):
            js = []
            for p in range(P):
                for r in range(E):
                    e = k * E + r
                    if e < len(rs[p]): js.append(rs[p][e])
            tot += len(set(j >> 3 for j in js)); ninst += 1; entries += len(js)
    return tot / entries * 32, entries / ninst
for P, E in ((32, 1), (16, 2), (8, 4), (4, 8)):
    lines, fill = cost(P, E)
    print(f"{P} particles x {E} lanes: lines per 32 gathered entries {lines:.2f}, lanes busy {fill:.1f}/32")
