"""Verlet build timing on cfg2 (BJ configs[1]): CUDA events around `reps`
pm_build_verlet calls (cells + list; each call synchronises) and, separately,
the list kernel alone through the step loop's rebuild.  PM_VERLET_STAGED=0
selects the previous (direct-store) builder.  Usage:
python tools/exp_build.py [--reps 20] [--dump out.npz]"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1804_07598_b200 import build, inputs, pm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--dump", default="")
ap.add_argument("--cfg", default="cfg2")
a = ap.parse_args()
build.build()
s = getattr(inputs, a.cfg)()
stream = torch.cuda.Stream()
c = pm.Context(stream=stream.cuda_stream)
c.set_domain(s.lo, s.hi, s.periodic)
c.set_cutoff(2.5, 0.3)
c.set_lj(1.0, 1.0, 1.0, 0.0)
c.place(s.pos, s.vel, s.gid)
c.build_verlet()
c.step_vv(0.005, 30)  # liquid-like state
for _ in range(3):
    c.build_verlet()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(stream)
for _ in range(a.reps):
    c.build_verlet()
e1.record(stream)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
cnt = c.count()
print(f"staged={os.environ.get('PM_VERLET_STAGED', '1')} build+cells {ms:.4f} ms, "
      f"nnz {cnt['nnz']} mean {cnt['nnz'] / s.n:.2f}")
if a.dump:
    rp, col = c.get_verlet()
    st = c.get_state()
    cnt = np.diff(rp)
    bad = None
    if os.path.exists(a.dump + ".npz"):  # compare with the other builder's dump
        o = np.load(a.dump + ".npz")
        og = dict(zip(o["gid"].tolist(), range(len(o["gid"]))))
        d = np.nonzero(cnt != o["cnt"][[og[g] for g in st["gid"].tolist()]])[0]
        print("rows with different counts:", d.size)
        for r in d[:5]:
            mine = set(col[rp[r]:rp[r + 1]].tolist())
            q = og[int(st["gid"][r])]
            other = set(o["col"][o["rp"][q]:o["rp"][q + 1]].tolist())
            print(" row", r, "gid", st["gid"][r], "pos", st["pos"][r], "only here", mine - other,
                  "only there", other - mine)
            from oracle import oracle
            for g2 in (mine ^ other):
                j = int(np.nonzero(st["gid"] == g2)[0][0])
                d2 = oracle.pair_d2(st["pos"][r, :3], st["pos"][j, :3], s.lo, s.hi, s.periodic)
                rv = np.float32(np.float32(2.5) + np.float32(0.3))
                print("   oracle d2", repr(d2), "rv2", repr(np.float32(rv * rv)),
                      "in" if d2 < np.float32(rv * rv) else "out",
                      st["pos"][r, :3].view(np.uint32), st["pos"][j, :3].view(np.uint32))
    else:
        np.savez(a.dump, rp=rp, col=col, gid=st["gid"], cnt=cnt)
