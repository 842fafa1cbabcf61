"""Experiment driver: run tools/prof_step.py-like cfg2 steps with an alternative
libpm.so (path in PM_LIB) and print the force-kernel time from the bench's
in-graph event profile.  An older library for the A/B: `git worktree add
/tmp/old <commit> && (cd /tmp/old && python -c "from paper_1804_07598_b200
import build; build.build()")`, then PM_LIB=/tmp/old/paper_1804_07598_b200/libpm.so."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_07598_b200 import inputs, pm  # noqa: E402

pm.lib(os.environ.get("PM_LIB", pm.LIB_PATH))
s = inputs.cfg2()
c = pm.Context()
c.set_domain(s.lo, s.hi, s.periodic)
c.set_cutoff(2.5, 0.3)
c.set_lj(1.0, 1.0, 1.0, 0.0)
c.place(s.pos, s.vel, s.gid)
c.step_vv(0.005, 60)
c.set_profiling(True)
r = c.step_vv(0.005, 300)
p = c.get_profile()
print(os.environ.get("PM_LIB", "default"), "force_us", 1e3 * p["force_ms"] / p["force_launches"],
      "step_us", 1e3 * p["step_ms"] / p["steps"], r)
