"""Profiling driver: cfg2 (BJ configs[1]) run through pm_step_vv WITHOUT CUDA
graphs (ncu cannot profile kernel nodes of graphs with conditional nodes), so
that `ncu -k regex:k_lj_step|k_verlet` sees the same kernels bench.py times
inside its graphs.  Usage: python tools/prof_step.py [--steps 40]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_07598_b200 import build, inputs, pm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=40)
ap.add_argument("--cfg", default="cfg2")
a = ap.parse_args()
build.build()
s = getattr(inputs, a.cfg)()
c = pm.Context(use_graphs=False)
c.set_domain(s.lo, s.hi, s.periodic)
c.set_cutoff(2.5, 0.3)
c.set_lj(1.0, 1.0, 1.0, 0.0)
c.place(s.pos, s.vel, s.gid)
r = c.step_vv(0.005, a.steps)
import json  # noqa: E402
print(json.dumps(r))
