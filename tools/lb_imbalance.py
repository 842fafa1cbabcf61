"""Load-balancing evidence for cfg5-class clustered inputs:
per-sub-domain pair work (list entries of the owned particles) of a 2x2x2
decomposition with equal cuboids vs the weighted-quantile tensor-product
cuts (dist.balanced_decomp).  Weights come from a one-context Verlet build.
Usage: python tools/lb_imbalance.py [--per-cluster 16384] [--clusters 64]"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_07598_b200 import build, dist, inputs, pm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--clusters", type=int, default=64)
ap.add_argument("--per-cluster", type=int, default=16384)
ap.add_argument("--sigma", type=float, default=4.0)
a = ap.parse_args()
build.build()
s = inputs.cfg5(n_clusters=a.clusters, per_cluster=a.per_cluster, sigma_c=a.sigma)
c = pm.Context()
c.set_domain(s.lo, s.hi, s.periodic)
c.set_cutoff(2.5, 0.3)
c.set_lj(1.0, 1.0, 1.0, 0.8)
c.place(s.pos, s.vel, s.gid)
c.build_verlet()
rp, _ = c.get_verlet(cols=False)
w = np.zeros(s.n)
w[c.get_state()["gid"]] = np.diff(rp)
c.close()
out = {"workload": f"cfg5-class: {a.clusters} Gaussian clusters x {a.per_cluster} "
                   f"(sigma_c={a.sigma}, mean rho 0.5), capped LJ r_min 0.8",
       "n": int(s.n), "pairs": float(w.sum())}
for grid in ((2, 1, 1), (2, 2, 1), (2, 2, 2)):
    Du = dist.Decomp(grid)
    Db = dist.balanced_decomp(grid, s.pos[:, :3], w, s.lo, s.hi, 2.8)
    res = {}
    for name, D in (("uniform", Du), ("balanced", Db)):
        own = dist.owner_of(s, D)
        work = np.bincount(own, weights=w, minlength=D.size)
        res[name] = {"imbalance_max_over_mean": dist.imbalance(work),
                     "work_per_rank": work.tolist()}
    res["cuts"] = [np.asarray(x).tolist() for x in Db.cuts]
    out["x".join(map(str, grid))] = res
print(json.dumps(out))


over = {}
for g in (2, 4, 6):
    grid = (g, g, g)
    for name, D in (("uniform", dist.Decomp(grid)),
                    ("balanced", dist.balanced_decomp(grid, s.pos[:, :3], w, s.lo, s.hi, 2.8))):
        own = dist.owner_of(s, D)
        work = np.bincount(own, weights=w, minlength=D.size)
        load = np.bincount(dist.lpt_assign(work, 8), weights=work, minlength=8)
        over[f"{g}x{g}x{g} {name} -> 8 ranks (LPT)"] = dist.imbalance(load)
print(json.dumps({"over_decomposition": over}))
