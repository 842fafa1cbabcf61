"""Loopback overhead of the native group path (pm_create_dist_local +
pm_dist_run) on ONE GPU: the cfg3 global system of grid g (one m^3 block per
sub-domain) run decomposed vs whole on one context, ms per step over K steps
(CUDA events on the shared stream), plus the sweep share (profiling pass).
Usage: python tools/exp_group_overhead.py [m] [K] [gx gy gz]
(GROUP_ONLY=1 / SINGLE_ONLY=1: one of the two runs)"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1804_07598_b200 import build, inputs, pm  # noqa: E402

build.build()
m = int(sys.argv[1]) if len(sys.argv) > 1 else 128
K = int(sys.argv[2]) if len(sys.argv) > 2 else 60
grid = tuple(int(x) for x in sys.argv[3:6]) if len(sys.argv) > 5 else (2, 1, 1)
s = inputs.cfg3_global(grid, m=m)
stream = torch.cuda.Stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(fn):
    torch.cuda.synchronize()
    e0.record(stream)
    t = time.perf_counter()
    r = fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), time.perf_counter() - t, r


ms1, r1 = float("nan"), {"rebuilds": -1}
if not os.environ.get("GROUP_ONLY"):
    c = pm.Context(stream=stream.cuda_stream)
    c.set_domain(s.lo, s.hi, s.periodic)
    c.set_cutoff(2.5, 0.3)
    c.set_lj(1.0, 1.0, 1.0, 0.0)
    c.place(s.pos, s.vel, s.gid)
    c.step_vv(0.005, 10)
    ms1, _, r1 = timed(lambda: c.step_vv(0.005, K))
    c.close()
    if os.environ.get("SINGLE_ONLY"):  # (for a launch list of the single context)
        print(f"one context {ms1 / K:.3f} ms/step ({r1['rebuilds']} rebuilds)")
        sys.exit(0)
mem = pm.create_dist_local(grid, stream=stream.cuda_stream)
for k, x in enumerate(mem):
    x.set_domain(s.lo, s.hi, s.periodic)
    x.set_cutoff(2.5, 0.3)
    x.set_lj(1.0, 1.0, 1.0, 0.0)
    x.place(s.pos if k == 0 else s.pos[:0], s.vel if k == 0 else s.vel[:0],
            s.gid if k == 0 else s.gid[:0])
for x in mem:
    x.map()
for x in mem:
    x.ghost_get()
for x in mem:
    x.dist_run(0.005, 10)
msg, wall, rg = timed(lambda: [x.dist_run(0.005, K) for x in mem][-1])
mem[0].set_profiling(True)
for x in mem:
    x.dist_run(0.005, 20)
pr = mem[0].get_profile()
mem[0].set_profiling(False)
print(f"grid {grid}, {s.n} particles: one context {ms1 / K:.3f} ms/step ({r1['rebuilds']} rebuilds);"
      f" group {msg / K:.3f} ms/step ({rg['rebuilds']} rebuilds, host wall {1e3 * wall / K:.3f})"
      f" ratio {msg / ms1:.3f}; sweeps {pr['force_ms'] / max(pr['force_launches'], 1):.3f} ms/step")
for x in mem:
    x.close()
