"""Measure the per-step cost of the decomposed driver (DistSim) against one
context on the same global system, on one GPU (loopback transport).  The
difference estimates the orchestration + exchange overhead per step."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1804_07598_b200 import dist, inputs, pm  # noqa: E402

grid = tuple(int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "2,1,1").split(","))
m = int(sys.argv[2]) if len(sys.argv) > 2 else 64
K = 200
s = inputs.cfg3_global(grid=grid, m=m)
# single context
c = pm.Context()
c.set_domain(s.lo, s.hi, s.periodic)
c.set_cutoff(2.5, 0.3)
c.set_lj(1.0, 1.0, 1.0, 0.0)
c.place(s.pos, s.vel, s.gid)
c.step_vv(0.005, 20)
torch.cuda.synchronize()
t0 = time.perf_counter()
r = c.step_vv(0.005, K)
torch.cuda.synchronize()
t_single = (time.perf_counter() - t0) / K
c.close()
# decomposed, loopback
D = dist.Decomp(grid)
owner = dist.owner_of(s, D)
stream = torch.cuda.Stream()
members = {q: dist.make_member(s.subset(np.where(owner == q)[0]), D, q, stream=stream)
           for q in range(D.size)}
sim = dist.DistSim(D, members, dist.LoopbackTransport(members), stream=stream)
sim.start()
sim.run(20)
torch.cuda.synchronize()
t0 = time.perf_counter()
reb = sim.run(K)
torch.cuda.synchronize()
t_dist = (time.perf_counter() - t0) / K
# refresh-only cost (no force): host + exchange
t0 = time.perf_counter()
for _ in range(50):
    sim.refresh()
torch.cuda.synchronize()
t_ref = (time.perf_counter() - t0) / 50
print(f"grid {grid} N={s.n}: single {1e3*t_single:.3f} ms/step ({r['rebuilds']} reb), "
      f"decomposed {1e3*t_dist:.3f} ms/step ({reb} reb), refresh {1e3*t_ref:.3f} ms")
