"""Experiment driver: pm_sph_run rate on cfg4 (BJ configs[3]) with the libpm.so
named by PM_LIB, plus the per-kernel profile of the stepping kernels."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_07598_b200 import inputs, pm  # noqa: E402

pm.lib(os.environ.get("PM_LIB", pm.LIB_PATH))
s = inputs.cfg4()
p = s.params
c = pm.Context()
c.set_domain(s.lo, s.hi, s.periodic)
c.set_cutoff(2.0 * p["h"], 0.1 * p["h"])
c.set_sph(p)
c.place(s.pos, s.vel, s.gid, s.kind)
c.build_verlet()
z = c.get_state()["pos"][:, 2].astype(np.float64)
P = p["rho0"] * 9.81 * np.maximum(p["h_swl"] - z, 0.0)
c.set_rho((p["rho0"] * (1.0 + P / p["b"]) ** (1.0 / p["gamma"])).astype(np.float32))
c.sph_run(10)
t0 = time.perf_counter()
r = c.sph_run(200)
t1 = time.perf_counter()
print(os.environ.get("PM_LIB", "default"),
      f"{1e3 * (t1 - t0) / r['steps']:.4f} ms/step rebuilds {r['rebuilds']} dt {r['dt_min']:.4e}")
print("stepping list entries per particle", c.count()["nnz"] / s.n)
