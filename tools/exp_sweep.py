"""A/B of the LJ step sweep on cfg2 (BJ configs[1]): ms per step over K
graph steps and the force-kernel time (CUDA events in the step graph), plus a
hash of the final positions (the staged and the int32 sweeps must agree bit
for bit).  PM_SWEEP_STAGED=0 selects the int32 gather sweep.
Usage: python tools/exp_sweep.py [K]"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1804_07598_b200 import build, inputs, pm  # noqa: E402

build.build()
K = int(sys.argv[1]) if len(sys.argv) > 1 else 300
s = inputs.cfg2()
stream = torch.cuda.Stream()
c = pm.Context(stream=stream.cuda_stream)
c.set_domain(s.lo, s.hi, s.periodic)
c.set_cutoff(2.5, 0.3)
c.set_lj(1.0, 1.0, 1.0, 0.0)
c.place(s.pos, s.vel, s.gid)
c.step_vv(0.005, 20)
h = hashlib.sha1(c.get_state()["pos"].tobytes()).hexdigest()[:12]
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(stream)
r = c.step_vv(0.005, K)
e1.record(stream)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / K
c.set_profiling(True)
c.step_vv(0.005, 100)
p = c.get_profile()
print(f"staged={os.environ.get('PM_SWEEP_STAGED', '1')} step {ms:.4f} ms, sweep "
      f"{p['force_ms'] / p['force_launches']:.4f} ms, rebuilds {r['rebuilds']}, "
      f"pos hash after 20 steps {h}")
