"""Workload for compute-sanitizer (memcheck / racecheck / synccheck): every
kernel family once on small inputs -- cfg1 (BJ configs[0]) and a 32^3 LJ
lattice through cell list + staged Verlet build + forces + 20 steps (graph and
plain launches), the half-list path, an SPH pass and run, a DEM run, and a
(2,1,1) loopback group (map, ghost_get, 10 steps).  Usage:
compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_1804_07598_b200 import build, inputs, pm  # noqa: E402

build.build()


def lj(s, use_graphs=True, newton=False):
    c = pm.Context(use_graphs=use_graphs)
    c.set_domain(s.lo, s.hi, s.periodic)
    c.set_cutoff(2.5, 0.3)
    c.set_lj(1.0, 1.0, 1.0, 0.0)
    if newton:
        c.set_newton(True)
    c.place(s.pos, s.vel, s.gid)
    c.build_verlet()
    c.compute_lj(want_energy=True)
    c.step_vv(0.005, 20)
    c.get_state()
    c.get_verlet()
    c.close()


lj(inputs.shuffled(inputs.cfg1(), (11,)))
s32 = inputs.lj_lattice_system(32, 32, 32, jitter_key=(3,), vel_key=(103,))
lj(s32)
lj(s32, use_graphs=False)
lj(s32, newton=True)
s4 = inputs.cfg4(dp=1.0 / 24.0, vel_key=(104,))
p = s4.params
c = pm.Context()
c.set_domain(s4.lo, s4.hi, s4.periodic)
c.set_cutoff(2.0 * p["h"], 0.1 * p["h"])
c.set_sph(p)
c.place(s4.pos, s4.vel, s4.gid, s4.kind)
c.build_verlet()
c.sph_density()
c.sph_forces()
c.sph_run(10)
c.close()
s5 = inputs.dem_avalanche(8, 6, 5)
q = s5.params
c = pm.Context()
c.set_domain(s5.lo, s5.hi, s5.periodic)
c.set_cutoff(2.0 * q["R"], q["skin"])
c.set_dem(q)
c.place(s5.pos, s5.vel, s5.gid)
c.dem_run(q["dt"], 30)
c.close()
g = inputs.cfg3_global((2, 1, 1), m=16)
mem = pm.create_dist_local((2, 1, 1))
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
    x.dist_run(0.005, 10)
for x in mem:
    x.close()
print("sanitize workload done")
