"""Profiling driver for the WCSPH pass (cfg4, BJ configs[3]): Verlet build with
r_v = 2h, density/EOS, forces -- run 3 times.  ncu -k regex:k_sph|k_verlet."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_07598_b200 import build, inputs, pm  # noqa: E402

build.build()
s = inputs.cfg4()
p = s.params
c = pm.Context()
c.set_domain(s.lo, s.hi, s.periodic)
c.set_cutoff(2.0 * p["h"], 0.0)
c.set_sph(p)
c.place(s.pos, s.vel, s.gid, s.kind)
for _ in range(3):
    c.build_verlet()
    c.sph_density()
    c.sph_forces()
print(c.count())
