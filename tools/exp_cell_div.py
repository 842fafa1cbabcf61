"""cfg2 velocity-Verlet steps with cell_div 1 vs 2 (reading R2): build and
step time from the context's event profile.  Usage: python tools/exp_cell_div.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_07598_b200 import inputs, pm  # noqa: E402

s = inputs.cfg2()
for cd in (1, 2):
    c = pm.Context(cell_div=cd)
    c.set_domain(s.lo, s.hi, s.periodic)
    c.set_cutoff(2.5, 0.3)
    c.set_lj(1.0, 1.0, 1.0, 0.0)
    c.place(s.pos, s.vel, s.gid)
    c.step_vv(0.005, 60)
    c.set_profiling(True)
    r = c.step_vv(0.005, 300)
    p = c.get_profile()
    print(f"cell_div={cd} force_us {1e3 * p['force_ms'] / p['force_launches']:.1f} "
          f"step_us {1e3 * p['step_ms'] / p['steps']:.1f} rebuilds {r['rebuilds']}")
    c.close()
