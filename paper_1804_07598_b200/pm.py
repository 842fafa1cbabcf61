"""Thin ctypes binding of include/pm.h (argument marshalling only).

Every step of the path runs in libpm.so's CUDA kernels; this module only
converts numpy arrays / torch CUDA tensors to pointers and status codes to
exceptions.  There is no CPU fallback: if libpm.so is missing or cannot be
loaded, ``lib()`` raises.
"""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpm.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "pm.h")

PM_OK = 0
PM_HOST, PM_DEVICE = 0, 1
STATUS = {0: "PM_OK", -1: "PM_E_INVAL", -2: "PM_E_STATE", -3: "PM_E_NOMEM", -4: "PM_E_CUDA",
          -5: "PM_E_NCCL", -6: "PM_E_DOMAIN", -7: "PM_E_COINCIDENT", -8: "PM_E_NONFINITE",
          -9: "PM_E_CAPACITY"}


class PMError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class Opts(C.Structure):
    _fields_ = [("device", C.c_int32), ("cell_div", C.c_int32), ("nbr_cap", C.c_int32),
                ("use_graphs", C.c_int32), ("cuda_stream", C.c_void_p)]


class SPHParams(C.Structure):
    _fields_ = [("h", C.c_float), ("mass", C.c_float), ("rho0", C.c_float), ("gamma", C.c_float),
                ("b", C.c_float), ("alpha", C.c_float), ("cbar", C.c_float), ("eta2", C.c_float),
                ("g", C.c_float * 3)]


class DEMParams(C.Structure):
    _fields_ = [("R", C.c_float), ("m", C.c_float), ("I", C.c_float), ("kn", C.c_float),
                ("kt", C.c_float), ("gamma_n", C.c_float), ("gamma_t", C.c_float),
                ("mu", C.c_float), ("g", C.c_float * 3), ("walls", C.c_int32 * 6)]


class SPHRunStats(C.Structure):
    _fields_ = [("steps", C.c_int64), ("rebuilds", C.c_int64), ("time", C.c_double),
                ("dt_min", C.c_float), ("dt_max", C.c_float), ("dt_last", C.c_float)]


class RunStats(C.Structure):
    _fields_ = [("steps", C.c_int64), ("rebuilds", C.c_int64), ("max_row", C.c_int32),
                ("nbr_cap", C.c_int32), ("mean_row", C.c_double)]


_lib = None
vp = C.c_void_p


def lib(path: str = None):
    """Load libpm.so (raises if it is missing -- the product has no fallback).
    PM_LIB=<path> loads another build of the same library (the bounds-checked
    libpm_checks.so of build.build(checks=True))."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("PM_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise RuntimeError(f"libpm.so not found at {path}; run __graft_entry__.build()")
    L = C.CDLL(path)
    st = C.c_int32
    sig = {
        "pm_opts_default": (st, [C.POINTER(Opts)]),
        "pm_version": (C.c_char_p, []),
        "pm_create": (st, [C.POINTER(Opts), C.POINTER(vp)]),
        "pm_destroy": (None, [vp]),
        "pm_last_error": (C.c_char_p, [vp]),
        "pm_set_domain": (st, [vp, vp, vp, vp]),
        "pm_set_cutoff": (st, [vp, C.c_float, C.c_float]),
        "pm_set_lj": (st, [vp, C.c_float, C.c_float, C.c_float, C.c_int32, C.c_float]),
        "pm_set_vlimit": (st, [vp, C.c_float]),
        "pm_set_sph": (st, [vp, C.POINTER(SPHParams)]),
        "pm_place": (st, [vp, C.c_int64, vp, vp, vp, vp, C.c_int32]),
        "pm_build_cells": (st, [vp]),
        "pm_build_verlet": (st, [vp]),
        "pm_compute_lj": (st, [vp, C.c_int32]),
        "pm_sph_density": (st, [vp]),
        "pm_sph_forces": (st, [vp]),
        "pm_sph_run": (st, [vp, C.c_int64, C.c_float, C.c_int32, C.POINTER(SPHRunStats)]),
        "pm_set_rho": (st, [vp, vp, C.c_int32]),
        "pm_set_dem": (st, [vp, C.POINTER(DEMParams)]),
        "pm_dem_run": (st, [vp, C.c_float, C.c_int64, vp]),
        "pm_get_dem": (st, [vp, vp, vp]),
        "pm_step_vv": (st, [vp, C.c_float, C.c_int64, C.POINTER(RunStats)]),
        "pm_count": (st, [vp, vp, vp, vp, vp]),
        "pm_get_cells": (st, [vp, vp, vp, vp]),
        "pm_get_verlet": (st, [vp, vp, vp]),
        "pm_get_state": (st, [vp, vp, vp, vp, vp, vp, vp, C.c_int32]),
        "pm_get_thermo": (st, [vp, vp, vp, vp, vp, vp]),
        "pm_get_kind": (st, [vp, vp]),
        "pm_thermo_compute": (st, [vp]),
        "pm_set_profiling": (st, [vp, C.c_int32]),
        "pm_get_profile": (st, [vp, vp, vp, vp, vp]),
        "pm_record_bytes": (C.c_int32, [C.c_int32]),
        "pm_set_decomposition": (st, [vp, vp, vp]),
        "pm_set_decomposition_cuts": (st, [vp, vp, vp, vp]),
        "pm_dist_plan": (st, [vp, C.c_int32, vp, vp]),
        "pm_dist_pack": (st, [vp, C.c_int32, vp]),
        "pm_dist_unpack": (st, [vp, C.c_int32, vp, C.c_int64]),
        "pm_dist_finish": (st, [vp]),
        "pm_dist_refresh_pack": (st, [vp, vp]),
        "pm_dist_refresh_unpack": (st, [vp, vp]),
        "pm_dist_step": (st, [vp, C.c_float, C.c_int32, vp]),
        "pm_set_newton": (st, [vp, C.c_int32]),
        "pm_get_verlet_shifts": (st, [vp, vp]),
        "pm_dist_read_flag": (st, [vp, vp]),
        "pm_dist_ghost_put_pack": (st, [vp, vp]),
        "pm_dist_ghost_put_unpack": (st, [vp, vp]),
        "pm_dist_pos_buffers": (st, [vp, vp, vp]),
        "pm_dist_ghost_slots": (st, [vp, vp]),
        "pm_dist_peer_setup": (st, [vp, C.c_int32, vp, vp, vp, vp]),
        "pm_dist_ipc_handles": (st, [vp, vp]),
        "pm_dist_ipc_open": (st, [vp, vp, vp, vp]),
        "pm_dist_ipc_close_all": (st, [vp]),
        "pm_dist_dem_init": (st, [vp]),
        "pm_dist_dem_step": (st, [vp, C.c_float, vp]),
        "pm_dist_refresh_pvw_pack": (st, [vp, vp]),
        "pm_dist_refresh_pvw_unpack": (st, [vp, vp]),
        "pm_dist_sph_init": (st, [vp]),
        "pm_dist_sph_rates": (st, [vp, vp]),
        "pm_dist_sph_update": (st, [vp, C.c_float, C.c_float, C.c_int32, vp]),
        "pm_dist_refresh_pv_pack": (st, [vp, vp]),
        "pm_dist_refresh_pv_unpack": (st, [vp, vp]),
        "pm_nccl_unique_id": (st, [vp]),
        "pm_create_dist": (st, [C.POINTER(Opts), C.c_int32, C.c_int32, vp, vp, C.POINTER(vp)]),
        "pm_create_dist_local": (st, [C.POINTER(Opts), vp, C.c_int32, vp]),
        "pm_dist_info": (st, [vp, vp, vp, vp, vp]),
        "pm_map": (st, [vp]),
        "pm_ghost_get": (st, [vp]),
        "pm_dist_run": (st, [vp, C.c_float, C.c_int64, C.POINTER(RunStats)]),
        "pm_dist_thermo": (st, [vp, vp, vp, vp, vp, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def header_symbols(header: str = HEADER):
    """Function names declared in include/pm.h."""
    txt = open(header).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(pm_[a-z_0-9]+)\s*\(", txt)))


def _ptr(a):
    """Pointer of a numpy array (host) or torch tensor (host or device)."""
    if a is None:
        return None, PM_HOST
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr()), (PM_DEVICE if a.is_cuda else PM_HOST)
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("arrays must be C-contiguous")
    return C.c_void_p(a.ctypes.data), PM_HOST


class Context:
    """One pm_ctx (one GPU, one stream)."""

    def __init__(self, device: int = 0, nbr_cap: int = 0, use_graphs=None, stream=None,
                 cell_div: int = 1, _handle=None):
        L = lib()
        o = Opts()
        L.pm_opts_default(C.byref(o))  # honours PM_USE_GRAPHS=0
        o.device = device
        o.nbr_cap = nbr_cap
        o.cell_div = cell_div
        if use_graphs is not None:
            o.use_graphs = 1 if use_graphs else 0
        o.cuda_stream = stream
        self.L = L
        self.n = 0
        if _handle is not None:  # a group member created by pm_create_dist[_local]
            self.h = _handle
            return
        h = vp()
        self._check(L.pm_create(C.byref(o), C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.L.pm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _check(self, code):
        if code != PM_OK:
            msg = lib().pm_last_error(self.h).decode() if getattr(self, "h", None) else ""
            raise PMError(code, msg)

    # ---- configuration
    def set_domain(self, lo, hi, periodic):
        lo = np.ascontiguousarray(lo, np.float32)
        hi = np.ascontiguousarray(hi, np.float32)
        per = np.ascontiguousarray(periodic, np.int32)
        self._check(self.L.pm_set_domain(self.h, lo.ctypes.data, hi.ctypes.data, per.ctypes.data))
        self._box = (lo.copy(), hi.copy())

    def set_cutoff(self, r_cut, skin):
        self._check(self.L.pm_set_cutoff(self.h, r_cut, skin))
        self._rv = float(np.float32(np.float32(r_cut) + np.float32(skin)))

    def set_lj(self, epsilon=1.0, sigma=1.0, mass=1.0, r_min=0.0):
        flags = PM_LJ_CAPPED if r_min > 0 else 0  # reading R22's capped force
        self._check(self.L.pm_set_lj(self.h, epsilon, sigma, mass, flags, r_min))

    def set_vlimit(self, vmax):
        self._check(self.L.pm_set_vlimit(self.h, vmax))

    def set_sph(self, p: dict):
        s = SPHParams(h=p["h"], mass=p["mass"], rho0=p["rho0"], gamma=p["gamma"], b=p["b"],
                      alpha=p["alpha"], cbar=p["c0"], eta2=p["eta2"])
        for d in range(3):
            s.g[d] = p["g"][d]
        self._check(self.L.pm_set_sph(self.h, C.byref(s)))

    # ---- data
    def place(self, pos4, vel4=None, gid=None, kind=None):
        n = int(pos4.shape[0])
        pp, mem = _ptr(pos4)
        pv, _ = _ptr(vel4)
        pg, _ = _ptr(gid)
        pk, _ = _ptr(kind)
        self._check(self.L.pm_place(self.h, n, pp, pv, pg, pk, mem))
        self.n = n

    def place_system(self, s):
        """Place an inputs.System and set its domain."""
        self.set_domain(s.lo, s.hi, s.periodic)
        self.place(s.pos, s.vel, s.gid, s.kind)

    def build_cells(self):
        self._check(self.L.pm_build_cells(self.h))

    def build_verlet(self):
        self._check(self.L.pm_build_verlet(self.h))

    def compute_lj(self, want_energy=False):
        self._check(self.L.pm_compute_lj(self.h, 1 if want_energy else 0))

    def sph_density(self):
        self._check(self.L.pm_sph_density(self.h))

    def sph_forces(self):
        self._check(self.L.pm_sph_forces(self.h))

    def set_newton(self, on: bool):
        """Half (Newton) lists with reductions for the j side (NEXT-1)."""
        self._check(self.L.pm_set_newton(self.h, 1 if on else 0))

    def set_dem(self, p):
        """p: dict with R, m, I, kn, kt, gn, gt, mu, g (3), walls (6 flags)."""
        d = DEMParams(float(p["R"]), float(p["m"]), float(p["I"]), float(p["kn"]),
                      float(p["kt"]), float(p["gn"]), float(p["gt"]), float(p["mu"]),
                      (C.c_float * 3)(*[float(x) for x in p["g"]]),
                      (C.c_int32 * 6)(*[int(x) for x in p["walls"]]))
        self._check(self.L.pm_set_dem(self.h, C.byref(d)))

    def dem_run(self, dt, nsteps):
        reb = C.c_int64(0)
        self._check(self.L.pm_dem_run(self.h, float(dt), int(nsteps), C.byref(reb)))
        return int(reb.value)

    def get_dem(self):
        c = self.count()
        n = c["n_owned"] + c["n_ghost"]  # local rows incl. ghost copies, as get_state
        w = np.zeros((n, 4), np.float32)
        t = np.zeros((n, 4), np.float32)
        self._check(self.L.pm_get_dem(self.h, w.ctypes.data, t.ctypes.data))
        return dict(omega=w, torque=t)

    def set_rho(self, rho):
        """Densities in the current internal order (as get_state returns them)."""
        r = np.ascontiguousarray(rho, dtype=np.float32)
        self._check(self.L.pm_set_rho(self.h, r.ctypes.data, PM_HOST))

    def sph_run(self, nsteps, cfl=0.2, every=40):
        """WCSPH time stepping (pm_sph_run): continuity density, Verlet scheme."""
        rs = SPHRunStats()
        self._check(self.L.pm_sph_run(self.h, int(nsteps), float(cfl), int(every), C.byref(rs)))
        return dict(steps=rs.steps, rebuilds=rs.rebuilds, time=rs.time, dt_min=rs.dt_min,
                    dt_max=rs.dt_max, dt_last=rs.dt_last)

    def step_vv(self, dt, nsteps):
        rs = RunStats()
        self._check(self.L.pm_step_vv(self.h, dt, int(nsteps), C.byref(rs)))
        return dict(steps=rs.steps, rebuilds=rs.rebuilds, max_row=rs.max_row,
                    nbr_cap=rs.nbr_cap, mean_row=rs.mean_row)

    # ---- getters
    def count(self):
        v = [C.c_int64() for _ in range(4)]
        self._check(self.L.pm_count(self.h, *[C.byref(x) for x in v]))
        return dict(n_owned=v[0].value, n_ghost=v[1].value, n_cells=v[2].value, nnz=v[3].value)

    def get_cells(self):
        c = self.count()
        n, nc = c["n_owned"], c["n_cells"]
        cell_of = np.zeros(n, np.int32)
        start = np.zeros(nc + 1, np.int32)
        perm = np.zeros(n, np.int32)
        self._check(self.L.pm_get_cells(self.h, cell_of.ctypes.data, start.ctypes.data,
                                        perm.ctypes.data))
        return dict(cell_of=cell_of, start=start, perm=perm)

    def get_verlet(self, cols=True):
        """CSR (row_ptr, col_gid) of the list; cols=False: row_ptr only."""
        c = self.count()
        n = c["n_owned"] + c["n_ghost"]  # one (possibly empty) row per local particle
        rp = np.zeros(n + 1, np.int64)
        self._check(self.L.pm_get_verlet(self.h, rp.ctypes.data, None))
        if not cols:
            return rp, None
        col = np.zeros(max(int(rp[-1]), 1), np.int64)
        self._check(self.L.pm_get_verlet(self.h, rp.ctypes.data, col.ctypes.data))
        return rp, col[:int(rp[-1])]

    def get_verlet_shifts(self):
        """(nnz, 3) int8 image shifts in get_verlet()'s order."""
        rp, _ = self.get_verlet(cols=False)
        sh = np.zeros((max(int(rp[-1]), 1), 3), np.int8)
        self._check(self.L.pm_get_verlet_shifts(self.h, sh.ctypes.data))
        return sh[:int(rp[-1])]

    def get_state(self):
        c = self.count()
        n = c["n_owned"] + c["n_ghost"]  # local particles incl. ghost copies
        pos = np.zeros((n, 4), np.float32)
        vel = np.zeros((n, 4), np.float32)
        f = np.zeros((n, 4), np.float32)
        gid = np.zeros(n, np.int64)
        rho = np.zeros(n, np.float32)
        pres = np.zeros(n, np.float32)
        self._check(self.L.pm_get_state(self.h, pos.ctypes.data, vel.ctypes.data, f.ctypes.data,
                                        gid.ctypes.data, rho.ctypes.data, pres.ctypes.data,
                                        PM_HOST))
        return dict(pos=pos, vel=vel, force=f, gid=gid, rho=rho, pres=pres)

    def get_state_into(self, pos4=None, vel4=None):
        """Copy pos/vel into caller buffers (numpy host or torch device)."""
        pp, mem = _ptr(pos4)
        pv, mem2 = _ptr(vel4)
        if pos4 is not None and vel4 is not None and mem != mem2:
            raise ValueError("pos4 and vel4 must both be host or both device")
        self._check(self.L.pm_get_state(self.h, pp, pv, None, None, None, None,
                                        mem if pos4 is not None else mem2))

    def kind(self):
        c = self.count()
        k = np.zeros(c["n_owned"] + c["n_ghost"], np.int32)
        self._check(self.L.pm_get_kind(self.h, k.ctypes.data))
        return k

    def thermo(self, recompute=True):
        if recompute:
            self._check(self.L.pm_thermo_compute(self.h))
        v = [C.c_double() for _ in range(4)]
        npairs = C.c_int64()
        self._check(self.L.pm_get_thermo(self.h, *[C.byref(x) for x in v], C.byref(npairs)))
        return dict(ke=v[0].value, pe_raw=v[1].value, pe_shift=v[2].value, virial=v[3].value,
                    npairs=npairs.value)

    def set_profiling(self, on: bool):
        self._check(self.L.pm_set_profiling(self.h, 1 if on else 0))

    def get_profile(self):
        fm, sm = C.c_double(), C.c_double()
        fl, ns = C.c_int64(), C.c_int64()
        self._check(self.L.pm_get_profile(self.h, C.byref(fm), C.byref(fl), C.byref(sm),
                                          C.byref(ns)))
        return dict(force_ms=fm.value, force_launches=fl.value, step_ms=sm.value, steps=ns.value)


PM_LJ_CAPPED = 1
PM_MSG_MIGRATE, PM_MSG_GHOST, PM_MSG_REFRESH, PM_MSG_REFRESH_PV = 0, 1, 2, 3
PM_MSG_REFRESH_PVW, PM_MSG_MIGRATE_HIST = 4, 5
PM_PHASE_PROLOGUE, PM_PHASE_STEP, PM_PHASE_FINAL, PM_PHASE_FORCES = 0, 1, 2, 3
PM_PHASE_NEWTON_FORCES, PM_PHASE_NEWTON_STEP, PM_PHASE_NEWTON_FINAL = 4, 5, 6
GHOST_BIT = 1 << 30


def record_bytes(what: int) -> int:
    return int(lib().pm_record_bytes(what))


def _dev_ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


class DistContext(Context):
    """A Context owning one cuboid of a decomposed periodic box (pm.h
    multi-GPU section); buffers are torch device tensors."""

    def set_decomposition(self, grid, coord):
        g = np.ascontiguousarray(grid, np.int32)
        c = np.ascontiguousarray(coord, np.int32)
        self._check(self.L.pm_set_decomposition(self.h, g.ctypes.data, c.ctypes.data))

    def set_decomposition_cuts(self, grid, coord, cuts):
        """cuts: per-axis sequences of interior cut positions (len grid[d]-1)."""
        g = np.ascontiguousarray(grid, np.int32)
        c = np.ascontiguousarray(coord, np.int32)
        flat = np.ascontiguousarray(np.concatenate([np.asarray(cuts[d], np.float32).reshape(-1)
                                                    for d in range(3)] + [np.zeros(1, np.float32)]))
        self._check(self.L.pm_set_decomposition_cuts(self.h, g.ctypes.data, c.ctypes.data,
                                                     flat.ctypes.data))

    def dist_plan(self, what, order):
        o = np.ascontiguousarray(order, np.int32)
        cnt = np.zeros(27, np.int64)
        self._check(self.L.pm_dist_plan(self.h, what, o.ctypes.data, cnt.ctypes.data))
        return cnt

    def dist_pack(self, what, send):
        self._check(self.L.pm_dist_pack(self.h, what, _dev_ptr(send)))

    def dist_unpack(self, what, recv, nrecv):
        self._check(self.L.pm_dist_unpack(self.h, what, _dev_ptr(recv), int(nrecv)))

    def dist_finish(self):
        self._check(self.L.pm_dist_finish(self.h))

    def refresh_pack(self, send, pv=False):
        """pv: False (positions), True / "pv" (+ velocities, SPH), "pvw"
        (+ angular velocities, DEM)."""
        f = {False: self.L.pm_dist_refresh_pack, True: self.L.pm_dist_refresh_pv_pack,
             "pv": self.L.pm_dist_refresh_pv_pack, "pvw": self.L.pm_dist_refresh_pvw_pack}[pv]
        self._check(f(self.h, _dev_ptr(send)))

    def refresh_unpack(self, recv, pv=False):
        f = {False: self.L.pm_dist_refresh_unpack, True: self.L.pm_dist_refresh_pv_unpack,
             "pv": self.L.pm_dist_refresh_pv_unpack,
             "pvw": self.L.pm_dist_refresh_pvw_unpack}[pv]
        self._check(f(self.h, _dev_ptr(recv)))

    def dist_dem_init(self):
        self._check(self.L.pm_dist_dem_init(self.h))

    def dist_dem_step(self, dt):
        f = C.c_int32(0)
        self._check(self.L.pm_dist_dem_step(self.h, float(dt), C.byref(f)))
        return int(f.value)

    def dist_sph_init(self):
        self._check(self.L.pm_dist_sph_init(self.h))

    def dist_sph_rates(self):
        b = C.c_float(0.0)
        self._check(self.L.pm_dist_sph_rates(self.h, C.byref(b)))
        return float(b.value)

    def dist_sph_update(self, bound, cfl=0.2, every=40):
        f = C.c_int32(0)
        self._check(self.L.pm_dist_sph_update(self.h, float(bound), float(cfl), int(every),
                                              C.byref(f)))
        return int(f.value)

    def get_kind(self):
        c = self.count()
        k = np.zeros(c["n_owned"] + c["n_ghost"], np.int32)
        self._check(self.L.pm_get_kind(self.h, k.ctypes.data))
        return k

    def owned_state(self):
        """get_state() restricted to owned particles (ghost copies removed)."""
        st = self.get_state()
        own = (self.get_kind() & GHOST_BIT) == 0
        return {k: v[own] for k, v in st.items()}

    def dist_step(self, dt, phase, read_flag=False):
        f = C.c_int32(0)
        self._check(self.L.pm_dist_step(self.h, dt, phase, C.byref(f) if read_flag else None))
        return int(f.value)

    def ghost_put_pack(self, send):
        self._check(self.L.pm_dist_ghost_put_pack(self.h, _dev_ptr(send)))

    def ghost_put_unpack(self, recv):
        self._check(self.L.pm_dist_ghost_put_unpack(self.h, _dev_ptr(recv)))

    def pos_buffers(self):
        a, b = vp(), vp()
        self._check(self.L.pm_dist_pos_buffers(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def ghost_slots(self, out):
        """Copy the ghost slots (arrival order) into the int32 device tensor out."""
        self._check(self.L.pm_dist_ghost_slots(self.h, _dev_ptr(out)))

    def peer_setup(self, peer_bufs, dst_peer, dst_slot):
        """peer_bufs: [(pos0, pos1)] device pointers per peer index; dst_peer /
        dst_slot: int32 device tensors over the ghost send list."""
        k = len(peer_bufs)
        p0 = (vp * max(k, 1))(*[b[0] for b in peer_bufs])
        p1 = (vp * max(k, 1))(*[b[1] for b in peer_bufs])
        self._check(self.L.pm_dist_peer_setup(self.h, k, p0, p1, _dev_ptr(dst_peer),
                                              _dev_ptr(dst_slot)))

    def ipc_handles(self):
        buf = (C.c_char * 128)()
        self._check(self.L.pm_dist_ipc_handles(self.h, buf))
        return bytes(buf)

    def ipc_open(self, handles: bytes):
        buf = (C.c_char * 128).from_buffer_copy(handles)
        a, b = vp(), vp()
        self._check(self.L.pm_dist_ipc_open(self.h, buf, C.byref(a), C.byref(b)))
        return a.value, b.value

    def ipc_close_all(self):
        self._check(self.L.pm_dist_ipc_close_all(self.h))

    def read_flag(self):
        f = C.c_int32(0)
        self._check(self.L.pm_dist_read_flag(self.h, C.byref(f)))
        return int(f.value)


# ---------------------------------------------------------------- groups (pm.h)
def _opts(device=0, stream=None, nbr_cap=0):
    o = Opts()
    lib().pm_opts_default(C.byref(o))
    o.device = device
    o.nbr_cap = nbr_cap
    o.cuda_stream = stream
    return o


def nccl_unique_id() -> bytes:
    """pm_nccl_unique_id: 128 bytes for rank 0 to broadcast."""
    buf = (C.c_char * 128)()
    code = lib().pm_nccl_unique_id(buf)
    if code != PM_OK:
        raise PMError(code, "pm_nccl_unique_id")
    return bytes(buf)


class GroupMember(DistContext):
    """A member of a multi-GPU group (pm_create_dist / pm_create_dist_local).
    map / ghost_get / dist_run / dist_thermo are collective: call them on
    every member (the last local member's call does the work)."""

    def map(self):
        self._check(self.L.pm_map(self.h))

    def ghost_get(self):
        self._check(self.L.pm_ghost_get(self.h))

    def dist_run(self, dt, nsteps):
        r = RunStats()
        self._check(self.L.pm_dist_run(self.h, float(dt), int(nsteps), C.byref(r)))
        return dict(steps=r.steps, rebuilds=r.rebuilds)

    def dist_thermo(self):
        v = [C.c_double(0.0) for _ in range(4)]
        npair = C.c_int64(0)
        self._check(self.L.pm_dist_thermo(self.h, *[C.byref(x) for x in v], C.byref(npair)))
        return dict(ke=v[0].value, pe_raw=v[1].value, pe_shift=v[2].value, virial=v[3].value,
                    npairs=int(npair.value))

    def dist_info(self):
        v = [C.c_int32(0) for _ in range(4)]
        self._check(self.L.pm_dist_info(self.h, *[C.byref(x) for x in v]))
        return dict(sub_domain=v[0].value, nsub=v[1].value, rank=v[2].value, nranks=v[3].value)


def create_dist(rank, nranks, uid: bytes, grid, device=0, stream=None, nbr_cap=0):
    """pm_create_dist: this process's member of an nranks-GPU group."""
    o = _opts(device, stream, nbr_cap)
    g = np.ascontiguousarray(grid, np.int32)
    idb = (C.c_char * 128).from_buffer_copy(uid)
    h = vp()
    code = lib().pm_create_dist(C.byref(o), int(rank), int(nranks), idb, g.ctypes.data,
                                C.byref(h))
    if code != PM_OK:
        raise PMError(code, "pm_create_dist")
    return GroupMember(device=device, stream=stream, _handle=h)


def create_dist_local(grid, device=0, stream=None, via_nccl=False, nbr_cap=0):
    """pm_create_dist_local: all sub-domains of `grid` in this process."""
    o = _opts(device, stream, nbr_cap)
    g = np.ascontiguousarray(grid, np.int32)
    P = int(np.prod(g))
    hs = (vp * P)()
    code = lib().pm_create_dist_local(C.byref(o), g.ctypes.data, 1 if via_nccl else 0, hs)
    if code != PM_OK:
        raise PMError(code, "pm_create_dist_local")
    return [GroupMember(device=device, stream=stream, _handle=vp(hs[k])) for k in range(P)]


def sorted_by_gid(state: dict) -> dict:
    """Reorder a get_state() dict into ascending gid order."""
    o = np.argsort(state["gid"], kind="stable")
    return {k: v[o] for k, v in state.items()}
