"""Long NVE runs of the fp32 path: total energy (kinetic + shifted LJ) every
`every` steps, on one context (cfg2, BJ configs[1]) and through the group API
in loopback (cfg3 (2,1,1), 2 x 2,097,152), with the relative drift
|E(t) - E(0)| / |E(0)| and the rebuild count.  The truncated (unshifted-force)
potential makes E drift slowly by itself; the same run on one context and on
the group shows the decomposition adds nothing to it.

Usage: python tools/nve_drift.py [steps] [every] > profiles/r02_nve_drift.json"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_07598_b200 import build, inputs, pm  # noqa: E402

build.build()
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
every = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
dt = 0.005


def energy(th):
    return th["ke"] + th["pe_shift"]


out = {"dt": dt, "steps": steps, "every": every}

s = inputs.cfg2()
c = pm.Context()
c.set_domain(s.lo, s.hi, s.periodic)
c.set_cutoff(2.5, 0.3)
c.set_lj(1.0, 1.0, 1.0, 0.0)
c.place(s.pos, s.vel, s.gid)
c.step_vv(dt, 1)
e0 = energy(c.thermo())
series, reb = [], 0
t0 = time.perf_counter()
for k in range(steps // every):
    r = c.step_vv(dt, every)
    reb += r["rebuilds"]
    e = energy(c.thermo())
    series.append({"step": (k + 1) * every, "E": e, "rel_drift": abs(e - e0) / abs(e0)})
out["cfg2_one_context"] = {"n": s.n, "E0": e0, "rebuilds": reb, "series": series,
                           "max_rel_drift": max(x["rel_drift"] for x in series),
                           "wall_s": time.perf_counter() - t0}
c.close()

grid = (2, 1, 1)
g = inputs.cfg3_global(grid)
res = {}
for label in ("one_context", "group_2x1x1"):
    if label == "one_context":
        ctx = pm.Context()
        ctx.set_domain(g.lo, g.hi, g.periodic)
        ctx.set_cutoff(2.5, 0.3)
        ctx.set_lj(1.0, 1.0, 1.0, 0.0)
        ctx.place(g.pos, g.vel, g.gid)
        ctx.step_vv(dt, 1)
        run = lambda n: ctx.step_vv(dt, n)  # noqa: E731
        th = lambda: ctx.thermo()  # noqa: E731
        closers = [ctx]
    else:
        mem = pm.create_dist_local(grid)
        for k, x in enumerate(mem):
            x.set_domain(g.lo, g.hi, g.periodic)
            x.set_cutoff(2.5, 0.3)
            x.set_lj(1.0, 1.0, 1.0, 0.0)
            x.place(g.pos if k == 0 else g.pos[:0], g.vel if k == 0 else g.vel[:0],
                    g.gid if k == 0 else g.gid[:0])
        for x in mem:
            x.map()
        for x in mem:
            x.ghost_get()
        for x in mem:
            x.dist_run(dt, 1)
        run = lambda n: [x.dist_run(dt, n) for x in mem][-1]  # noqa: E731
        th = lambda: [x.dist_thermo() for x in mem][-1]  # noqa: E731
        closers = mem
    e0 = energy(th())
    series, reb = [], 0
    nsteps = steps // 4
    for k in range(nsteps // every):
        r = run(every)
        reb += r["rebuilds"]
        e = energy(th())
        series.append({"step": (k + 1) * every, "E": e, "rel_drift": abs(e - e0) / abs(e0)})
    res[label] = {"E0": e0, "rebuilds": reb, "series": series,
                  "max_rel_drift": max(x["rel_drift"] for x in series)}
    for x in closers:
        x.close()
out["cfg3_2x1x1"] = {"n": g.n, **res}
print(json.dumps(out, indent=1))
