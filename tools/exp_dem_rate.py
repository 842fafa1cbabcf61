"""Experiment driver: pm_dem_run rate on the DEM avalanche (inputs.dem_avalanche)
with the libpm.so named by PM_LIB (CUDA events around 500 steps after 300)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1804_07598_b200 import inputs, pm  # noqa: E402

pm.lib(os.environ.get("PM_LIB", pm.LIB_PATH))
s = inputs.dem_avalanche()
p = s.params
st = torch.cuda.Stream()
c = pm.Context(stream=st.cuda_stream)
c.set_domain(s.lo, s.hi, s.periodic)
c.set_cutoff(2.0 * p["R"], p["skin"])
c.set_dem(p)
c.place(s.pos, s.vel, s.gid)
c.dem_run(p["dt"], 300)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(st)
reb = c.dem_run(p["dt"], 500)
e1.record(st)
torch.cuda.synchronize()
print(os.environ.get("PM_LIB", "default"), f"{e0.elapsed_time(e1) / 500:.4f} ms/step rebuilds {reb}")
