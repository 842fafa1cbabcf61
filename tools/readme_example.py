"""The README usage example, runnable: cfg2, 1000 velocity-Verlet steps."""
import sys; sys.path.insert(0, '.')
from paper_1804_07598_b200 import build, inputs, pm
build.build()
s = inputs.cfg2()
c = pm.Context()
c.set_domain(s.lo, s.hi, s.periodic)
c.set_cutoff(2.5, 0.3)
c.set_lj(1.0, 1.0, 1.0, 0.0)
c.place(s.pos, s.vel, s.gid)
print(c.step_vv(0.005, 1000))
