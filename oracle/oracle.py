"""TEST INFRASTRUCTURE ONLY -- the CPU oracle (ctypes over liboracle.so).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.  It never imports the
product package's binding and shares no arithmetic with the CUDA path; the
only shared module is the seeded input generator
(paper_1804_07598_b200/inputs.py), which holds none of the method.

Every function cites the PAPER.md passage it follows; the definitions live in
oracle/pm_oracle.c.  Pins: tests/test_oracle_pins.py.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "pm_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared", "-fPIC",
          "-std=c11", "-Wall"]


def build(force: bool = False) -> str:
    """Compile oracle/pm_oracle.c -> oracle/liboracle.so with gcc."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, SRC, "-lm"])
        os.replace(tmp, LIB)
    return LIB


_lib = None

f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
i8p = np.ctypeslib.ndpointer(np.int8, flags="C_CONTIGUOUS")


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        L.orc_num_threads.restype = C.c_int
        L.orc_set_num_threads.argtypes = [C.c_int]
        L.orc_wrap.restype = C.c_int64
        L.orc_wrap.argtypes = [C.c_int64, f32p, f32p, f32p, i32p]
        L.orc_cell_grid.restype = C.c_int
        L.orc_cell_grid.argtypes = [f32p, f32p, C.c_float, C.c_int32, i32p, f32p]
        L.orc_cell_ids.argtypes = [C.c_int64, f32p, f32p, f32p, i32p, i32p]
        L.orc_counting_sort.argtypes = [C.c_int64, i32p, C.c_int64, i32p, i32p, i32p]
        L.orc_pair_d2.restype = C.c_float
        L.orc_pair_d2.argtypes = [f32p, f32p, f32p, f32p, i32p]
        L.orc_verlet_rows.restype = C.c_int64
        L.orc_verlet_rows.argtypes = [C.c_int64, f32p, f32p, f32p, i32p, C.c_float, i64p,
                                      C.c_int64, i64p, i32p, C.c_void_p, C.c_int64]
        L.orc_lj_rows.restype = C.c_int64
        L.orc_lj_rows.argtypes = [C.c_int64, f32p, f32p, f32p, i32p, C.c_float, C.c_double,
                                  C.c_double, C.c_double, i64p, C.c_int64, f64p, f64p, f64p,
                                  i64p]
        L.orc_lj_V.restype = C.c_double
        L.orc_lj_V.argtypes = [C.c_double] * 3
        L.orc_lj_mdVdr.restype = C.c_double
        L.orc_lj_mdVdr.argtypes = [C.c_double] * 3
        L.orc_vv_run.argtypes = [C.c_int64, f64p, f64p, f64p, f64p, i32p, C.c_double,
                                 C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
                                 C.c_int64, f64p]
        L.orc_sph_W.restype = C.c_double
        L.orc_sph_W.argtypes = [C.c_double, C.c_double]
        L.orc_sph_dWdr.restype = C.c_double
        L.orc_sph_dWdr.argtypes = [C.c_double, C.c_double]
        L.orc_sph_density_rows.argtypes = [C.c_int64, f32p, f32p, f32p, i32p, C.c_double,
                                           C.c_double, C.c_double, C.c_double, C.c_double,
                                           i64p, C.c_int64, f64p, f64p]
        L.orc_sph_accel_rows.argtypes = [C.c_int64, f32p, f32p, f64p, f64p, C.c_void_p, f32p,
                                         f32p, i32p, C.c_double, C.c_double, C.c_double,
                                         C.c_double, C.c_double, f64p, i64p, C.c_int64, f64p]
        L.orc_dem_run.restype = C.c_int64
        L.orc_dem_run.argtypes = [C.c_int64, f64p, f64p, f64p, i64p, f64p, f64p, i32p, i32p,
                                  C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
                                  C.c_double, C.c_double, C.c_double, f64p, C.c_double,
                                  C.c_int64, C.c_int64]
        L.orc_sph_run.argtypes = [C.c_int64, f64p, f64p, f64p, C.c_void_p, f64p, f64p, i32p,
                                  C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
                                  C.c_double, C.c_double, C.c_double, f64p, C.c_double,
                                  C.c_int64, C.c_int64, f64p]
        L.orc_md_cells_run.restype = C.c_int64
        L.orc_md_cells_run.argtypes = [C.c_int64, f64p, f64p, f64p, f64p, i32p, C.c_double,
                                       C.c_double, C.c_double, C.c_double, C.c_double,
                                       C.c_double, C.c_double, C.c_int64, C.c_void_p]
        _lib = L
    return _lib


def num_threads() -> int:
    return int(lib().orc_num_threads())


def set_num_threads(n: int) -> None:
    lib().orc_set_num_threads(int(n))


def _f3(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32).reshape(3))


def _i3(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32).reshape(3))


def _rows(rows, n):
    if rows is None:
        return np.arange(n, dtype=np.int64)
    return np.ascontiguousarray(np.asarray(rows, dtype=np.int64))


# ---------------------------------------------------------------- cell list
def wrap(pos4, lo, hi, per):
    """R1 fp32 wrap (PAPER.md:166 periodic BCs).  Returns (wrapped copy, #bad)."""
    p = np.ascontiguousarray(pos4, dtype=np.float32).copy()
    bad = lib().orc_wrap(p.shape[0], p, _f3(lo), _f3(hi), _i3(per))
    return p, int(bad)


def cell_grid(lo, hi, rv, cell_div=1):
    """R2 (PAPER.md:48 Cell Lists).  Returns (ncell int32[3], inv_w float32[3])."""
    nc = np.zeros(3, np.int32)
    iw = np.zeros(3, np.float32)
    lib().orc_cell_grid(_f3(lo), _f3(hi), np.float32(rv), int(cell_div), nc, iw)
    return nc, iw


def cell_list(pos4, lo, hi, per, rv, cell_div=1):
    """R1-R3 + step 5: wrap, cell ids, counts, start, stable perm."""
    p, bad = wrap(pos4, lo, hi, per)
    nc, iw = cell_grid(lo, hi, rv, cell_div)
    n = p.shape[0]
    cell_of = np.zeros(n, np.int32)
    lib().orc_cell_ids(n, p, _f3(lo), iw, nc, cell_of)
    ncell = int(nc[0]) * int(nc[1]) * int(nc[2])
    count = np.zeros(ncell, np.int32)
    start = np.zeros(ncell + 1, np.int32)
    perm = np.zeros(n, np.int32)
    lib().orc_counting_sort(n, cell_of, ncell, count, start, perm)
    return dict(pos=p, bad=bad, ncell=nc, inv_w=iw, cell_of=cell_of, count=count, start=start,
                perm=perm)


def pair_d2(xi, xj, lo, hi, per) -> np.float32:
    """R4 fp32 pair distance^2 (pinned decision function)."""
    return np.float32(lib().orc_pair_d2(_f3(xi), _f3(xj), _f3(lo), _f3(hi), _i3(per)))


# ---------------------------------------------------------------- Verlet
def verlet_rows(pos4, lo, hi, per, rv, rows=None, want_shift=True):
    """R5: N_i = {j != i : d2_32 < rv^2} by brute force (PAPER.md:164 Verlet
    lists; PAPER.md:48 O(N^2) definition).  Returns (row_ptr, cols, shifts)."""
    p = np.ascontiguousarray(pos4, dtype=np.float32)
    n = p.shape[0]
    r = _rows(rows, n)
    rp = np.zeros(r.shape[0] + 1, np.int64)
    cap = max(1, 128 * r.shape[0])
    while True:
        cols = np.zeros(cap, np.int32)
        sh = np.zeros(3 * cap, np.int8) if want_shift else None
        tot = lib().orc_verlet_rows(n, p, _f3(lo), _f3(hi), _i3(per), np.float32(rv), r,
                                    r.shape[0], rp, cols,
                                    sh.ctypes.data if sh is not None else None, cap)
        if tot >= 0:
            break
        cap = -tot
    cols = cols[:tot]
    sh = sh[:3 * tot].reshape(-1, 3) if sh is not None else None
    return rp, cols, sh


# ---------------------------------------------------------------- LJ
def lj_V(r, eps=1.0, sigma=1.0):
    """PAPER.md:162 V_LJ(r) = 4 eps [(sigma/r)^12 - (sigma/r)^6]."""
    return lib().orc_lj_V(float(r), float(eps), float(sigma))


def lj_mdVdr(r, eps=1.0, sigma=1.0):
    """-dV/dr of PAPER.md:162 (reading R7)."""
    return lib().orc_lj_mdVdr(float(r), float(eps), float(sigma))


def lj_rows(pos4, lo, hi, per, rc, eps=1.0, sigma=1.0, r_min=0.0, rows=None):
    """LJ forces/energies per row, fp64 values, R6 fp32 inclusion.
    Returns dict(F (nrows,3), U, W, npair, ncoinc)."""
    p = np.ascontiguousarray(pos4, dtype=np.float32)
    n = p.shape[0]
    r = _rows(rows, n)
    m = r.shape[0]
    F = np.zeros((m, 3), np.float64)
    U = np.zeros(m, np.float64)
    W = np.zeros(m, np.float64)
    npair = np.zeros(m, np.int64)
    nco = lib().orc_lj_rows(n, p, _f3(lo), _f3(hi), _i3(per), np.float32(rc), float(eps),
                            float(sigma), float(r_min), r, m, F, U, W, npair)
    return dict(F=F, U=U, W=W, npair=npair, ncoinc=int(nco))


def vv_run(pos4, vel4, lo, hi, per, rc, dt, nsteps, eps=1.0, sigma=1.0, mass=1.0, r_min=0.0):
    """fp64 velocity-Verlet trajectory (Listing 4.1 at
    PAPER.md:291-293, 320).  Returns (x, v, trace[nsteps+1, 4]) with trace
    columns KE, U_raw, U_shift, npairs."""
    x = np.ascontiguousarray(np.asarray(pos4)[:, :3], dtype=np.float64).copy()
    v = np.ascontiguousarray(np.asarray(vel4)[:, :3], dtype=np.float64).copy()
    n = x.shape[0]
    tr = np.zeros((nsteps + 1) * 4, np.float64)
    lo64 = np.ascontiguousarray(np.asarray(lo, np.float32).astype(np.float64))
    hi64 = np.ascontiguousarray(np.asarray(hi, np.float32).astype(np.float64))
    lib().orc_vv_run(n, x.reshape(-1), v.reshape(-1), lo64, hi64, _i3(per), float(rc),
                     float(eps), float(sigma), float(r_min), float(mass), float(dt),
                     int(nsteps), tr)
    return x, v, tr.reshape(nsteps + 1, 4)


def md_cells_run(pos4, vel4, lo, hi, per, rc, skin, dt, nsteps, eps=1.0, sigma=1.0, mass=1.0,
                 r_min=0.0, trace=True):
    """The method itself on the CPU (SURVEY §8(d) oracle timing): fp64 cell
    list + Verlet list with skin (rebuild at skin/2) + velocity Verlet
    (Listing 4.1 at PAPER.md:291-320).  Same
    trajectory as vv_run up to summation order.  Returns (x, v, trace or
    None, number of list builds)."""
    x = np.ascontiguousarray(np.asarray(pos4)[:, :3], dtype=np.float64).copy()
    v = np.ascontiguousarray(np.asarray(vel4)[:, :3], dtype=np.float64).copy()
    n = x.shape[0]
    tr = np.zeros((nsteps + 1) * 4, np.float64) if trace else None
    lo64 = np.ascontiguousarray(np.asarray(lo, np.float32).astype(np.float64))
    hi64 = np.ascontiguousarray(np.asarray(hi, np.float32).astype(np.float64))
    nb = lib().orc_md_cells_run(n, x.reshape(-1), v.reshape(-1), lo64, hi64, _i3(per),
                                float(rc), float(skin), float(eps), float(sigma), float(r_min),
                                float(mass), float(dt), int(nsteps),
                                tr.ctypes.data if tr is not None else None)
    if nb < 0:
        raise ValueError("md_cells_run: a periodic axis has fewer than 3 cells of side r_v")
    return x, v, (tr.reshape(nsteps + 1, 4) if tr is not None else None), int(nb)


# ---------------------------------------------------------------- SPH
def sph_W(r, h):
    """Cubic spline kernel (PAPER.md:342 'classic cubic SPH kernel [34]')."""
    return lib().orc_sph_W(float(r), float(h))


def sph_dWdr(r, h):
    return lib().orc_sph_dWdr(float(r), float(h))


def sph_density_rows(pos4, lo, hi, per, params, rows=None):
    """Density summation (reading R16) + Tait EOS Eq. 3.
    Returns (rho, P) fp64 for the rows."""
    p = np.ascontiguousarray(pos4, dtype=np.float32)
    n = p.shape[0]
    r = _rows(rows, n)
    rho = np.zeros(r.shape[0], np.float64)
    P = np.zeros(r.shape[0], np.float64)
    lib().orc_sph_density_rows(n, p, _f3(lo), _f3(hi), _i3(per), float(params["h"]),
                               float(params["mass"]), float(params["rho0"]),
                               float(params["b"]), float(params["gamma"]), r, r.shape[0],
                               rho, P)
    return rho, P


def sph_accel_rows(pos4, vel4, rho, P, kind, lo, hi, per, params, rows=None):
    """Eq. 1 momentum equation with Eq. 5 viscosity,
    readings R17-R20.  rho, P: fp64 per particle in storage order."""
    p = np.ascontiguousarray(pos4, dtype=np.float32)
    v = np.ascontiguousarray(vel4, dtype=np.float32)
    n = p.shape[0]
    r = _rows(rows, n)
    a = np.zeros((r.shape[0], 3), np.float64)
    k = None if kind is None else np.ascontiguousarray(kind, dtype=np.int32)
    g = np.ascontiguousarray(np.asarray(params["g"], np.float64).reshape(3))
    lib().orc_sph_accel_rows(n, p, v, np.ascontiguousarray(rho, dtype=np.float64),
                             np.ascontiguousarray(P, dtype=np.float64),
                             k.ctypes.data if k is not None else None, _f3(lo), _f3(hi),
                             _i3(per), float(params["h"]), float(params["mass"]),
                             float(params["alpha"]), float(params["c0"]),
                             float(params["eta2"]), g, r, r.shape[0], a)
    return a


def sph_run(pos4, vel4, rho, kind, lo, hi, per, params, nsteps, cfl=0.2, every=40):
    """WCSPH time stepping (SURVEY NEXT-3; PAPER.md:335 Eq. 2, :358 'Verlet
    time-stepping [46] with dynamic step size'; readings R26-R28): continuity
    density, Tait EOS, Eq. 1 + Eq. 5 accelerations, Verlet scheme with an
    Euler step every `every` steps, dt = cfl * min(dt_f, dt_cv).  fp64 state
    from the fp32 inputs.  Returns (x (n,3), v (n,3), rho (n,), dt (nsteps,))."""
    n = pos4.shape[0]
    x = np.ascontiguousarray(np.asarray(pos4, np.float32)[:, :3].astype(np.float64))
    v = np.ascontiguousarray(np.asarray(vel4, np.float32)[:, :3].astype(np.float64))
    r = np.ascontiguousarray(np.asarray(rho, np.float64).copy())
    k = None if kind is None else np.ascontiguousarray(kind, dtype=np.int32)
    g = np.ascontiguousarray(np.asarray(params["g"], np.float64).reshape(3))
    lo64 = np.ascontiguousarray(np.asarray(lo, np.float32).astype(np.float64))
    hi64 = np.ascontiguousarray(np.asarray(hi, np.float32).astype(np.float64))
    tr = np.zeros(max(int(nsteps), 1), np.float64)
    lib().orc_sph_run(n, x.reshape(-1), v.reshape(-1), r, k.ctypes.data if k is not None else None,
                      lo64, hi64, _i3(per), float(params["h"]), float(params["mass"]),
                      float(params["rho0"]), float(params["b"]), float(params["gamma"]),
                      float(params["alpha"]), float(params["c0"]), float(params["eta2"]), g,
                      float(cfl), int(every), int(nsteps), tr)
    return x, v, r, tr[:nsteps]


def dem_run(pos4, vel4, omega, gid, lo, hi, per, walls, params, dt, nsteps):
    """DEM (Eqs. 9-13; readings R29-R33):
    Hertzian normal force with damping, tangential spring with history and
    Coulomb cap, torques, planar walls, leapfrog.  fp64 state from the fp32
    inputs; O(N^2).  Returns (x, v, w (n,3) fp64, number of contacts)."""
    x = np.ascontiguousarray(np.asarray(pos4, np.float32)[:, :3].astype(np.float64))
    v = np.ascontiguousarray(np.asarray(vel4, np.float32)[:, :3].astype(np.float64))
    w = np.ascontiguousarray(np.asarray(omega, np.float32)[:, :3].astype(np.float64))
    n = x.shape[0]
    g = np.ascontiguousarray(np.asarray(params["g"], np.float64).reshape(3))
    lo64 = np.ascontiguousarray(np.asarray(lo, np.float32).astype(np.float64))
    hi64 = np.ascontiguousarray(np.asarray(hi, np.float32).astype(np.float64))
    nh = lib().orc_dem_run(n, x.reshape(-1), v.reshape(-1), w.reshape(-1),
                           np.ascontiguousarray(gid, dtype=np.int64), lo64, hi64, _i3(per),
                           np.ascontiguousarray(walls, dtype=np.int32), float(params["R"]),
                           float(params["m"]), float(params["I"]), float(params["kn"]),
                           float(params["kt"]), float(params["gn"]), float(params["gt"]),
                           float(params["mu"]), g, float(dt), int(nsteps), 64 * n + 64)
    return x, v, w, int(nh)


# ---------------------------------------------------------------- parity metric
def normalized_max_err(got, ref):
    """BJ north_star: max per-component |got - ref| / RMS(ref over all comps)."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    rms = float(np.sqrt(np.mean(ref * ref)))
    return float(np.max(np.abs(got - ref))) / (rms if rms > 0 else 1.0)
