"""Diagnostics for pm_sph_run: GPU vs oracle errors on a small dam break, and
the stepping rate on cfg4 (BJ configs[3]).  Usage: python tools/sph_run_check.py"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_07598_b200 import build, inputs, pm  # noqa: E402
from oracle import oracle  # noqa: E402

build.build()


def hydrostatic_rho(z, p):
    P = p["rho0"] * 9.81 * np.maximum(p["h_swl"] - np.asarray(z, np.float64), 0.0)
    return (p["rho0"] * (1.0 + P / p["b"]) ** (1.0 / p["gamma"])).astype(np.float32)


s = inputs.cfg4(dp=1.0 / 16.0)
p = s.params
c = pm.Context()
c.set_domain(s.lo, s.hi, s.periodic)
c.set_cutoff(2.0 * p["h"], 0.1 * p["h"])
c.set_sph(p)
c.place(s.pos, s.vel, s.gid, s.kind)
rho_init = hydrostatic_rho(s.pos[:, 2], p).astype(np.float64)
for nsteps in (30, 300):
    c.place(s.pos, s.vel, s.gid, s.kind)
    c.build_verlet()
    c.set_rho(hydrostatic_rho(c.get_state()["pos"][:, 2], p))
    r = c.sph_run(nsteps, cfl=0.2, every=10)
    st = c.get_state()
    o = np.argsort(st["gid"])
    x_ref, v_ref, rho_ref, dt_ref = oracle.sph_run(s.pos, s.vel, rho_init, s.kind, s.lo, s.hi,
                                                   s.periodic, p, nsteps, cfl=0.2, every=10)
    x = st["pos"][o, :3].astype(np.float64)
    v = st["vel"][o, :3].astype(np.float64)
    rho = st["rho"][o].astype(np.float64)
    print(f"n={s.n} steps={nsteps} rebuilds={r['rebuilds']} time={r['time']:.6e} "
          f"(ref {dt_ref.sum():.6e}) dx/dp={np.max(np.abs(x - x_ref)) / p['dp']:.2e} "
          f"dv/vmax={np.max(np.abs(v - v_ref)) / np.max(np.abs(v_ref)):.2e} "
          f"vmax={np.max(np.abs(v_ref)):.3e} drho/rho0={np.max(np.abs(rho - rho_ref)) / 1000:.2e}")
c.close()
# throughput on cfg4
s = inputs.cfg4()
p = s.params
c = pm.Context()
c.set_domain(s.lo, s.hi, s.periodic)
c.set_cutoff(2.0 * p["h"], 0.1 * p["h"])
c.set_sph(p)
c.place(s.pos, s.vel, s.gid, s.kind)
c.build_verlet()
c.set_rho(hydrostatic_rho(c.get_state()["pos"][:, 2], p))
c.sph_run(10)
t0 = time.perf_counter()
r = c.sph_run(100)
t1 = time.perf_counter()
print(f"cfg4 n={s.n}: {r['steps']} steps in {t1 - t0:.3f} s = {1e3 * (t1 - t0) / r['steps']:.3f} "
      f"ms/step, {s.n * r['steps'] / (t1 - t0):.3e} particle-steps/s, rebuilds {r['rebuilds']}, "
      f"dt {r['dt_min']:.3e}..{r['dt_max']:.3e}")
