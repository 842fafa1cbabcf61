"""DEM avalanche (inputs.dem_avalanche, 679,140 grains) for profiling:
`warm` steps, then `steps` steps.  Run under ncu with PM_USE_GRAPHS=0."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_07598_b200 import inputs, pm  # noqa: E402

warm = int(sys.argv[1]) if len(sys.argv) > 1 else 300
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
pm.lib(os.environ.get("PM_LIB", pm.LIB_PATH))
s = inputs.dem_avalanche()
p = s.params
c = pm.Context()
c.set_domain(s.lo, s.hi, s.periodic)
c.set_cutoff(2.0 * p["R"], p["skin"])
c.set_dem(p)
c.place(s.pos, s.vel, s.gid)
c.dem_run(p["dt"], warm)
print("rebuilds", c.dem_run(p["dt"], steps), "nnz/n", c.count()["nnz"] / s.n)
