"""Seeded synthetic inputs shared by the CUDA path, the oracle and the bench.

This module holds NO arithmetic of the method (no wrap rule, no cell ids, no
distances, no forces).  It only draws lattices, jitter, Maxwell velocities and
Gaussian clusters, in fp64, and rounds them once to fp32.  Both sides
(`oracle/` and the C-ABI library) consume exactly the arrays produced here.

Recipes follow SURVEY.md §8(d) and the readings R10-R14, R21-R23 listed in
DESIGN.md.  Every generator is keyed by a tuple fed to
``numpy.random.SeedSequence`` so that the same key always gives the same bytes.

Paper context: the MD client starts "on a regular Cartesian 60^3 mesh"
(§4.1) and the SPH client is a dam break "starting from a column
of fluid in the left corner of the domain" (§4.2, Fig. 5).  The
configurations themselves are BASELINE.json `configs[0..4]`.
"""
from __future__ import annotations

import dataclasses
import numpy as np

# Lattice constant of a simple-cubic lattice at reduced density 0.8 (BJ configs).
A_RHO08 = 0.8 ** (-1.0 / 3.0)


def rng(*key: int) -> np.random.Generator:
    """PCG64 generator for an integer key tuple."""
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(list(key))))


@dataclasses.dataclass
class System:
    """One particle system in storage order.

    pos, vel: float32 (n, 4); the 4th lane is 0 (padding for 16-byte loads).
    gid: int64 (n,), unique.  kind: int32 (n,) or None (0 fluid/LJ, 1 fixed
    boundary).  lo, hi: float32 (3,).  periodic: int32 (3,).
    """

    pos: np.ndarray
    vel: np.ndarray
    gid: np.ndarray
    lo: np.ndarray
    hi: np.ndarray
    periodic: np.ndarray
    kind: np.ndarray | None = None
    params: dict = dataclasses.field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.pos.shape[0])

    def subset(self, idx: np.ndarray) -> "System":
        return System(
            pos=np.ascontiguousarray(self.pos[idx]),
            vel=np.ascontiguousarray(self.vel[idx]),
            gid=np.ascontiguousarray(self.gid[idx]),
            lo=self.lo.copy(), hi=self.hi.copy(), periodic=self.periodic.copy(),
            kind=None if self.kind is None else np.ascontiguousarray(self.kind[idx]),
            params=dict(self.params))


def _as_pos4(xyz: np.ndarray) -> np.ndarray:
    out = np.zeros((xyz.shape[0], 4), dtype=np.float32)
    out[:, :3] = xyz.astype(np.float32)
    return out


def sc_lattice(nx: int, ny: int, nz: int, a: float, jitter: float, key, origin=(0.0, 0.0, 0.0)):
    """Simple-cubic lattice x = origin + (i + 0.5) a + U(-jitter, jitter), x fastest.

    Reading R12: jitter is uniform per coordinate, drawn in fp64,
    then the position is rounded once to fp32.  Returns (xyz float64 (n,3),
    lattice index (n,3) int64).
    """
    ix, iy, iz = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    # x fastest: order (iz, iy, ix)
    idx = np.stack([ix.transpose(2, 1, 0).ravel(), iy.transpose(2, 1, 0).ravel(),
                    iz.transpose(2, 1, 0).ravel()], axis=1).astype(np.int64)
    xyz = (idx.astype(np.float64) + 0.5) * a + np.asarray(origin, dtype=np.float64)
    if jitter > 0:
        xyz = xyz + rng(*key).uniform(-jitter, jitter, size=xyz.shape)
    return xyz, idx


def maxwell(n: int, T: float, mass: float, key) -> np.ndarray:
    """Maxwell velocities, reading R11: N(0, sqrt(T/m)) per component, mean
    removed, rescaled so that sum(m v^2) / (3n - 3) == T, rounded to fp32."""
    v = rng(*key).normal(0.0, np.sqrt(T / mass), size=(n, 3))
    v -= v.mean(axis=0)
    t_now = mass * float((v * v).sum()) / (3 * n - 3)
    v *= np.sqrt(T / t_now)
    return _as_pos4(v)


def lj_lattice_system(nx, ny, nz, jitter_key, vel_key=None, T=1.0, a=A_RHO08, jitter=0.05,
                      origin_cells=(0, 0, 0), box_cells=None) -> System:
    """LJ fluid on an SC lattice at rho = 0.8 (BJ configs[0..2]); periodic box
    [0, box_cells * a).  gid = ix + nx_box (iy + ny_box iz) in global lattice
    coordinates so that blocks of a decomposed system get disjoint gids."""
    if box_cells is None:
        box_cells = (nx, ny, nz)
    origin = tuple(c * a for c in origin_cells)
    xyz, idx = sc_lattice(nx, ny, nz, a, jitter, jitter_key, origin)
    gidx = idx + np.asarray(origin_cells, dtype=np.int64)
    gid = gidx[:, 0] + box_cells[0] * (gidx[:, 1] + box_cells[1] * gidx[:, 2])
    n = xyz.shape[0]
    vel = maxwell(n, T, 1.0, vel_key) if vel_key is not None else np.zeros((n, 4), np.float32)
    hi = np.array([box_cells[0] * a, box_cells[1] * a, box_cells[2] * a], dtype=np.float32)
    return System(pos=_as_pos4(xyz), vel=vel, gid=gid.astype(np.int64),
                  lo=np.zeros(3, np.float32), hi=hi, periodic=np.ones(3, np.int32),
                  params=dict(epsilon=1.0, sigma=1.0, mass=1.0, r_cut=2.5, skin=0.3, dt=0.005))


def cfg1() -> System:
    """BJ configs[0]: 4096 particles, 16^3 SC, jitter key (1,), zero velocity."""
    return lj_lattice_system(16, 16, 16, jitter_key=(1,))


def cfg2(nx=128, ny=128, nz=64) -> System:
    """BJ configs[1]: 1,048,576 particles; reading R10: SC 128 x 128 x 64;
    jitter key (2,), Maxwell T = 1 key (102,)."""
    return lj_lattice_system(nx, ny, nz, jitter_key=(2,), vel_key=(102,))


def cfg3_block(bx, by, bz, grid=(1, 1, 1), m=128) -> System:
    """BJ configs[2] per-GPU block: SC m^3 offset by m a (bx,by,bz);
    jitter key (3,bx,by,bz), velocities key (103,bx,by,bz) (per-block mean
    removal and T = 1 rescale).  Box = grid * m cells."""
    box = (grid[0] * m, grid[1] * m, grid[2] * m)
    return lj_lattice_system(m, m, m, jitter_key=(3, bx, by, bz), vel_key=(103, bx, by, bz),
                             origin_cells=(bx * m, by * m, bz * m), box_cells=box)


def cfg3_global(grid=(1, 1, 1), m=128) -> System:
    """All blocks of cfg3 concatenated (block order x fastest): the same global
    system at every decomposition."""
    parts = [cfg3_block(bx, by, bz, grid, m) for bz in range(grid[2])
             for by in range(grid[1]) for bx in range(grid[0])]
    s = parts[0]
    return System(pos=np.concatenate([p.pos for p in parts]),
                  vel=np.concatenate([p.vel for p in parts]),
                  gid=np.concatenate([p.gid for p in parts]),
                  lo=s.lo, hi=s.hi, periodic=s.periodic, params=s.params)


# SPH constants, readings R19-R21; PAPER.md:338-350 (§4.2 Eqs. 3-5).
SPH_RHO0 = 1000.0
SPH_GAMMA = 7.0
SPH_COEF_SOUND = 20.0
SPH_G = 9.81


def cfg4(dp=1.0 / 160.0, fluid=(1.0, 1.0, 0.5), box=(1.6, 1.0, 0.7), layers=3, vel_key=None,
         vmax=0.1) -> System:
    """BJ configs[3]: WCSPH dam-break-class block (readings R13, R14).

    Fluid lattice (i + 0.5) dp filling [0, fluid); 3 layers of fixed boundary
    particles on the x and y walls and the bottom (open top), over the full
    box height.  kind = 0 fluid, 1 boundary.  v = 0 unless vel_key is given
    (then U(-vmax, vmax) per component on fluid particles, to exercise Eq. 5).
    """
    nfx, nfy, nfz = (int(round(f / dp)) for f in fluid)
    nbx, nby, nbz = (int(round(b / dp)) for b in box)
    ix = np.arange(-layers, nbx + layers)
    iy = np.arange(-layers, nby + layers)
    iz = np.arange(-layers, nbz)
    IZ, IY, IX = np.meshgrid(iz, iy, ix, indexing="ij")
    IX, IY, IZ = IX.ravel(), IY.ravel(), IZ.ravel()
    wall = (IX < 0) | (IX >= nbx) | (IY < 0) | (IY >= nby) | (IZ < 0)
    fl = (IX >= 0) & (IX < nfx) & (IY >= 0) & (IY < nfy) & (IZ >= 0) & (IZ < nfz)
    keep = wall | fl
    IX, IY, IZ, wall = IX[keep], IY[keep], IZ[keep], wall[keep]
    xyz = (np.stack([IX, IY, IZ], axis=1).astype(np.float64) + 0.5) * dp
    n = xyz.shape[0]
    kind = wall.astype(np.int32)
    vel = np.zeros((n, 4), np.float32)
    if vel_key is not None:
        v = rng(*vel_key).uniform(-vmax, vmax, size=(n, 3))
        v[kind == 1] = 0.0
        vel[:, :3] = v.astype(np.float32)
    gid = np.arange(n, dtype=np.int64)
    lo = np.array([-layers * dp, -layers * dp, -layers * dp], dtype=np.float32)
    hi = np.array([box[0] + layers * dp, box[1] + layers * dp, box[2]], dtype=np.float32)
    h = 1.3 * dp
    h_swl = fluid[2]
    c0 = SPH_COEF_SOUND * np.sqrt(SPH_G * h_swl)
    params = dict(dp=dp, h=h, mass=SPH_RHO0 * dp ** 3, rho0=SPH_RHO0, gamma=SPH_GAMMA,
                  c0=c0, b=c0 * c0 * SPH_RHO0 / SPH_GAMMA, g=(0.0, 0.0, -SPH_G), h_swl=h_swl,
                  alpha=0.1, eta2=0.01 * h * h)
    return System(pos=_as_pos4(xyz), vel=vel, gid=gid, lo=lo, hi=hi,
                  periodic=np.zeros(3, np.int32), kind=kind, params=params)


def cfg5(n_clusters=64, per_cluster=131072, sigma_c=4.0, rho=0.5, key=5) -> System:
    """BJ configs[4]: Gaussian clusters (reading R22).
    Centres U[0, L)^3 with L = (N / rho)^(1/3); offsets N(0, sigma_c^2);
    positions wrapped into [0, L) in fp64 (np.mod) before the fp32 rounding;
    a value that rounds up to L is set to 0."""
    n = n_clusters * per_cluster
    L = (n / rho) ** (1.0 / 3.0)
    centres = rng(key).uniform(0.0, L, size=(n_clusters, 3))
    xyz = np.empty((n, 3), np.float64)
    for c in range(n_clusters):
        off = rng(key, c).normal(0.0, sigma_c, size=(per_cluster, 3))
        xyz[c * per_cluster:(c + 1) * per_cluster] = centres[c] + off
    xyz = np.mod(xyz, L)
    x32 = xyz.astype(np.float32)
    L32 = np.float32(L)
    x32[x32 >= L32] = 0.0
    pos = np.zeros((n, 4), np.float32)
    pos[:, :3] = x32
    vel = maxwell(n, 1.0, 1.0, (105,))
    return System(pos=pos, vel=vel, gid=np.arange(n, dtype=np.int64),
                  lo=np.zeros(3, np.float32), hi=np.full(3, L32, np.float32),
                  periodic=np.ones(3, np.int32),
                  params=dict(epsilon=1.0, sigma=1.0, mass=1.0, r_cut=2.5, skin=0.3, dt=0.005,
                              r_min=0.8))


def shuffled(s: System, key) -> System:
    """Random storage order (exercises the stable sort)."""
    perm = rng(*key).permutation(s.n)
    return s.subset(perm)


def random_box(n: int, L: float, key, periodic=(1, 1, 1)) -> System:
    """Uniform random points in [0, L)^3 (small brute-force cases)."""
    xyz = rng(*key).uniform(0.0, L, size=(n, 3))
    x32 = xyz.astype(np.float32)
    x32[x32 >= np.float32(L)] = 0.0
    pos = np.zeros((n, 4), np.float32)
    pos[:, :3] = x32
    return System(pos=pos, vel=np.zeros((n, 4), np.float32), gid=np.arange(n, dtype=np.int64),
                  lo=np.zeros(3, np.float32), hi=np.full(3, np.float32(L)),
                  periodic=np.asarray(periodic, np.int32),
                  params=dict(epsilon=1.0, sigma=1.0, mass=1.0, r_cut=2.5, skin=0.3, dt=0.005))


DEM_G = 9.81


def dem_avalanche(nx=147, ny=105, nz=44, incline_deg=30.0, key=(71,), vjit=0.01,
                  gap=1e-3) -> System:
    """DEM avalanche down an inclined plane (§4.5, Figs. 10-11;
    reading R34 in DESIGN.md): grains of radius R = 0.06 on a Cartesian
    lattice of spacing a = 2R (1 + 1e-3) (no initial overlap) filling
    [0, nx a) x [0, ny a) x [0, nz a); the default 147 x 105 x 44 = 679,140
    grains stand in for the paper's 677,310 with the aspect of its
    4.26 x 3.06 x 1.26 start box.  The domain stretches that box by the
    paper's 8.4/4.26 in x and 3.18/1.26 in z; walls at both x faces and the
    floor, free +z, periodic y (length ny a); gravity rotated by the
    incline about y.  Velocities U(-vjit, vjit) break the lattice symmetry.
    params: the Silbert constants of P:540 (k_n, k_t read x1000, R34) and
    mu = 0.5, gamma_t = 0 (R31-R32), dt = 2e-4, skin = 0.02.  `gap` widens the
    lattice spacing to 2R (1 + gap) (loose starts for the multi-GPU tests)."""
    R = 0.06
    a = 2.0 * R * (1.0 + gap)
    g = np.stack(np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"), -1)
    xyz = (g.reshape(-1, 3).astype(np.float64) + 0.5) * a
    n = xyz.shape[0]
    vel = np.zeros((n, 4), np.float32)
    vel[:, :3] = rng(*key).uniform(-vjit, vjit, (n, 3)).astype(np.float32)
    lo = np.zeros(3, np.float32)
    hi = np.array([nx * a * 8.4 / 4.26, ny * a, nz * a * 3.18 / 1.26], np.float32)
    th = np.deg2rad(incline_deg)
    params = dict(R=R, m=1.0, I=1.44e-3, kn=7849.0, kt=2243.0, gn=3.401, gt=0.0, mu=0.5,
                  g=(DEM_G * np.sin(th), 0.0, -DEM_G * np.cos(th)), walls=(1, 1, 0, 0, 1, 0),
                  dt=2e-4, skin=0.02)
    return System(pos=_as_pos4(xyz), vel=vel, gid=np.arange(n, dtype=np.int64), lo=lo, hi=hi,
                  periodic=np.array([0, 1, 0], np.int32), params=params)


def sph_layer(dp=1.0 / 160.0, nx=24, ny=24, nz=8, layers=3, vel_key=(106,), vmax=0.1) -> System:
    """A WCSPH fluid layer periodic in x and y (NEXT-3 multi-GPU stepping
    cases: decomposed axes must be periodic): fluid lattice (i + 0.5) dp on
    nx x ny x nz, `layers` fixed boundary layers below it, open top; the same
    constants as cfg4 with h_swl = nz dp; fluid velocities U(-vmax, vmax) key
    vel_key (0 if None)."""
    ix, iy, iz = np.arange(nx), np.arange(ny), np.arange(-layers, nz)
    IZ, IY, IX = np.meshgrid(iz, iy, ix, indexing="ij")
    xyz = (np.stack([IX.ravel(), IY.ravel(), IZ.ravel()], axis=1).astype(np.float64) + 0.5) * dp
    kind = (IZ.ravel() < 0).astype(np.int32)
    n = xyz.shape[0]
    vel = np.zeros((n, 4), np.float32)
    if vel_key is not None:
        v = rng(*vel_key).uniform(-vmax, vmax, size=(n, 3))
        v[kind == 1] = 0.0
        vel[:, :3] = v.astype(np.float32)
    lo = np.array([0.0, 0.0, -layers * dp], np.float32)
    hi = np.array([nx * dp, ny * dp, (nz + 6) * dp], np.float32)
    h = 1.3 * dp
    h_swl = nz * dp
    c0 = SPH_COEF_SOUND * np.sqrt(SPH_G * h_swl)
    params = dict(dp=dp, h=h, mass=SPH_RHO0 * dp ** 3, rho0=SPH_RHO0, gamma=SPH_GAMMA,
                  c0=c0, b=c0 * c0 * SPH_RHO0 / SPH_GAMMA, g=(0.0, 0.0, -SPH_G), h_swl=h_swl,
                  alpha=0.1, eta2=0.01 * h * h)
    return System(pos=_as_pos4(xyz), vel=vel, gid=np.arange(n, dtype=np.int64), lo=lo, hi=hi,
                  periodic=np.array([1, 1, 0], np.int32), kind=kind, params=params)
