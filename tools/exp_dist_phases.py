"""Host-side phase timing of DistSim (loopback, one GPU): wraps the driver's
phases with perf_counter accumulators (GPU synchronised around each phase)."""
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1804_07598_b200 import dist, inputs, pm  # noqa: E402

grid = tuple(int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "2,1,1").split(","))
m = int(sys.argv[2]) if len(sys.argv) > 2 else 128
s = inputs.cfg3_global(grid=grid, m=m)
D = dist.Decomp(grid)
owner = dist.owner_of(s, D)
stream = torch.cuda.Stream()
members = {q: dist.make_member(s.subset(np.where(owner == q)[0]), D, q, stream=stream)
           for q in range(D.size)}
sim = dist.DistSim(D, members, dist.LoopbackTransport(members), stream=stream)
acc = collections.defaultdict(float)
cnt = collections.Counter()


def wrap(obj, name):
    f = getattr(obj, name)

    def g(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize()
        acc[name] += time.perf_counter() - t0
        cnt[name] += 1
        return r
    setattr(obj, name, g)


sim.start()
sim.run(10)
for nm in ["_rebuild", "_refresh", "_message_round"]:
    wrap(sim, nm)
for ctx in members.values():
    for nm in ["dist_step", "dist_plan", "dist_pack", "dist_unpack", "dist_finish"]:
        wrap(ctx, nm)
torch.cuda.synchronize()
t0 = time.perf_counter()
sim.run(100)
torch.cuda.synchronize()
tot = time.perf_counter() - t0
print(f"total {1e3*tot:.1f} ms for 100 steps")
for k in sorted(acc, key=lambda k: -acc[k]):
    print(f"{k:16s} n={cnt[k]:5d} total={1e3*acc[k]:8.2f} ms mean={1e3*acc[k]/cnt[k]:.3f} ms")
