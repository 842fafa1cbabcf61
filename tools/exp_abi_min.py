"""Minimal-ABI timing of cfg2 steps for A/B runs against older library builds
(declares only the calls it uses, so a libpm.so from an earlier commit
loads).  Usage: PM_LIB=path python tools/exp_abi_min.py; build the older
library in a worktree: `git worktree add /tmp/old <commit>` and
`build.build()` there (exp_libs/ is only a scratch place for such copies)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_07598_b200 import inputs  # noqa: E402
from paper_1804_07598_b200.pm import Opts, RunStats  # noqa: E402

L = C.CDLL(os.environ["PM_LIB"])
vp = C.c_void_p
for name, args in {"pm_opts_default": [vp], "pm_create": [vp, vp], "pm_set_domain": [vp, vp, vp, vp],
                   "pm_set_cutoff": [vp, C.c_float, C.c_float],
                   "pm_set_lj": [vp, C.c_float, C.c_float, C.c_float, C.c_int32, C.c_float],
                   "pm_place": [vp, C.c_int64, vp, vp, vp, vp, C.c_int32],
                   "pm_step_vv": [vp, C.c_float, C.c_int64, vp], "pm_set_profiling": [vp, C.c_int32],
                   "pm_get_profile": [vp, vp, vp, vp, vp]}.items():
    getattr(L, name).argtypes = args
    getattr(L, name).restype = C.c_int32
s = inputs.cfg2()
o = Opts()
L.pm_opts_default(C.byref(o))
h = vp()
assert L.pm_create(C.byref(o), C.byref(h)) == 0
f = lambda a, t=np.float32: np.ascontiguousarray(a, t)
lo, hi, per = f(s.lo), f(s.hi), f(s.periodic, np.int32)
assert L.pm_set_domain(h, lo.ctypes.data, hi.ctypes.data, per.ctypes.data) == 0
assert L.pm_set_cutoff(h, 2.5, 0.3) == 0
assert L.pm_set_lj(h, 1.0, 1.0, 1.0, 0, 0.0) == 0
pos, vel, gid = f(s.pos), f(s.vel), f(s.gid, np.int64)
assert L.pm_place(h, s.n, pos.ctypes.data, vel.ctypes.data, gid.ctypes.data, None, 0) == 0
rs = RunStats()
assert L.pm_step_vv(h, 0.005, 60, C.byref(rs)) == 0
L.pm_set_profiling(h, 1)
assert L.pm_step_vv(h, 0.005, 300, C.byref(rs)) == 0
fm, fl, sm, ns = C.c_double(), C.c_int64(), C.c_double(), C.c_int64()
L.pm_get_profile(h, C.byref(fm), C.byref(fl), C.byref(sm), C.byref(ns))
print(os.environ["PM_LIB"], "force_us %.1f step_us %.1f rebuilds %d" %
      (1e3 * fm.value / fl.value, 1e3 * sm.value / ns.value, rs.rebuilds))
