"""Experiment driver: one WCSPH pass on cfg4 (build + density + forces, as the
bench's sph line) with the libpm.so named by PM_LIB, CUDA events over 10 passes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1804_07598_b200 import inputs, pm  # noqa: E402

pm.lib(os.environ.get("PM_LIB", pm.LIB_PATH))
s = inputs.cfg4()
p = s.params
st = torch.cuda.Stream()
c = pm.Context(stream=st.cuda_stream)
c.set_domain(s.lo, s.hi, s.periodic)
c.set_cutoff(2.0 * p["h"], 0.0)
c.set_sph(p)
c.place(s.pos, s.vel, s.gid, s.kind)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
tot = [0.0, 0.0, 0.0]
for it in range(12):
    torch.cuda.synchronize()
    ev[0].record(st)
    c.build_verlet()
    ev[1].record(st)
    c.sph_density()
    ev[2].record(st)
    c.sph_forces()
    ev[3].record(st)
    torch.cuda.synchronize()
    if it >= 2:
        for k in range(3):
            tot[k] += ev[k].elapsed_time(ev[k + 1]) / 10
print(os.environ.get("PM_LIB", "default"), "build %.3f density %.3f forces %.3f ms" % tuple(tot))
