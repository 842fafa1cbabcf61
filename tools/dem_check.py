"""Diagnostics for pm_dem_run vs the fp64 oracle (oracle.dem_run): a small
granular packing with walls, gravity and friction.  Prints max deviations
after a few horizons.  Usage: python tools/dem_check.py"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_07598_b200 import build, inputs, pm  # noqa: E402
from oracle import oracle  # noqa: E402

P = dict(R=0.06, m=1.0, I=1.44e-3, kn=7849.0, kt=2243.0, gn=3.401, gt=0.0, mu=0.5,
         g=(0.0, 0.0, -9.81), walls=(1, 1, 0, 0, 1, 0))


def granular(nx=10, ny=10, nz=8, a=0.125, key=(61,)):
    g = np.stack(np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"), -1)
    xyz = 0.07 + a * g.reshape(-1, 3).astype(np.float64)
    xyz[:, 2] += 0.02
    n = xyz.shape[0]
    pos = np.zeros((n, 4), np.float32)
    pos[:, :3] = xyz.astype(np.float32)
    vel = np.zeros((n, 4), np.float32)
    vel[:, :3] = inputs.rng(*key).uniform(-0.2, 0.2, (n, 3)).astype(np.float32)
    lo = np.array([0.0, 0.0, 0.0], np.float32)
    hi = np.array([nx * a + 0.02, ny * a, max(3.0, nz * a + 1.0)], np.float32)
    return pos, vel, np.arange(n, dtype=np.int64), lo, hi, np.array([0, 1, 0], np.int32)


if __name__ == "__main__":
    build.build()
    pos, vel, gid, lo, hi, per = granular()
    for nsteps in (200, 1000):
        c = pm.Context()
        c.set_domain(lo, hi, per)
        c.set_cutoff(2 * P["R"], 0.02)
        c.set_dem(P)
        c.place(pos, vel, gid)
        t0 = time.perf_counter()
        reb = c.dem_run(2e-4, nsteps)
        t1 = time.perf_counter()
        st = c.get_state()
        dm = c.get_dem()
        o = np.argsort(st["gid"])
        x_ref, v_ref, w_ref, nh = oracle.dem_run(pos, vel, np.zeros_like(pos), gid, lo, hi, per,
                                                 P["walls"], P, 2e-4, nsteps)
        x = st["pos"][o, :3].astype(np.float64)
        v = st["vel"][o, :3].astype(np.float64)
        w = dm["omega"][o, :3].astype(np.float64)
        print(f"n={len(gid)} steps={nsteps} rebuilds={reb} contacts={nh} "
              f"dx/R={np.max(np.abs(x - x_ref)) / P['R']:.2e} "
              f"dv/vmax={np.max(np.abs(v - v_ref)) / np.max(np.abs(v_ref)):.2e} "
              f"dw/wmax={np.max(np.abs(w - w_ref)) / max(np.max(np.abs(w_ref)), 1e-12):.2e} "
              f"wmax={np.max(np.abs(w_ref)):.3e} gpu {1e3 * (t1 - t0) / nsteps:.3f} ms/step")
        c.close()
    # throughput: a 1M-grain bed (lattice 100^3 at 2.08 R spacing), 200 steps
    pos, vel, gid, lo, hi, per = granular(100, 100, 100)
    c = pm.Context()
    c.set_domain(lo, hi, per)
    c.set_cutoff(2 * P["R"], 0.02)
    c.set_dem(P)
    c.place(pos, vel, gid)
    c.dem_run(2e-4, 20)
    t0 = time.perf_counter()
    reb = c.dem_run(2e-4, 200)
    t1 = time.perf_counter()
    print(f"dem bed n={len(gid)}: {1e3 * (t1 - t0) / 200:.3f} ms/step = "
          f"{len(gid) * 200 / (t1 - t0):.3e} particle-steps/s, rebuilds {reb}")
