"""NEXT-1 measurement: cfg2 (BJ configs[1]) velocity-Verlet steps with full
lists vs half (Newton) lists; force-phase time per step from the step graph's
event nodes (full: k_lj_step; Newton: clear F + k_lj_half + k_lj_half_vv) and
the whole step.  Usage: python tools/exp_newton.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_07598_b200 import inputs, pm  # noqa: E402

s = inputs.cfg2()
for newton in (False, True, False, True):
    c = pm.Context()
    c.set_newton(newton)
    c.set_domain(s.lo, s.hi, s.periodic)
    c.set_cutoff(2.5, 0.3)
    c.set_lj(1.0, 1.0, 1.0, 0.0)
    c.place(s.pos, s.vel, s.gid)
    c.step_vv(0.005, 60)
    c.set_profiling(True)
    r = c.step_vv(0.005, 300)
    p = c.get_profile()
    nnz = c.count()["nnz"]
    print(f"newton={newton} force_us {1e3 * p['force_ms'] / p['force_launches']:.1f} "
          f"step_us {1e3 * p['step_ms'] / p['steps']:.1f} rebuilds {r['rebuilds']} "
          f"entries/particle {nnz / s.n:.2f}")
    c.close()
