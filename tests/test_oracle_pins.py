"""Pins of the CPU oracle against things other than itself (no GPU).

Each test fixes part of the oracle with a value the paper / mathematics fixes:
closed forms (golden files), finite-difference derivatives, lattice sums by
integer enumeration, invariants, symmetry, brute-force fp64 band checks, and
conservation laws.  A dropped term, wrong sign, wrong index or transposed
operand in oracle/pm_oracle.c fails at least one of these.
"""
import itertools
import math
import os

import numpy as np
import pytest

from paper_1804_07598_b200 import inputs

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden_rows(name):
    rows = []
    with open(os.path.join(GOLD, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line.split())
    return rows


# ------------------------------------------------------------------ LJ pair
def test_lj_golden_closed_forms(orc):
    """zero crossing at sigma, minimum -eps at 2^(1/6) sigma,
    SPEC.md:698 worked example (240 at r = sigma = 0.1)."""
    for eps, sig, r, V, F in (map(float, row) for row in _golden_rows("lj_closed_forms.txt")):
        assert orc.lj_V(r, eps, sig) == pytest.approx(V, abs=1e-12 * max(1.0, abs(V)))
        assert orc.lj_mdVdr(r, eps, sig) == pytest.approx(F, abs=1e-9 * max(1.0, abs(F)))


@pytest.mark.parametrize("r", [0.85, 0.95, 1.0, 1.05, 1.3, 1.5, 2.0, 2.4, 2.5])
def test_lj_force_is_minus_dV_dr(orc, r):
    """-dV/dr from a central finite difference of V (pins the force formula
    against the potential of PAPER.md:162, reading R7)."""
    h = 1e-5
    fd = -(orc.lj_V(r + h) - orc.lj_V(r - h)) / (2 * h)
    assert orc.lj_mdVdr(r) == pytest.approx(fd, rel=1e-7, abs=1e-8)


def test_lj_two_particle_spec_example(orc):
    """sigma = 0.1, eps = 1, r = sigma along x, q at +x:
    F_p = (-240, 0, 0), F_q = (+240, 0, 0); energy = V(sigma) = 0.  Also a
    two-particle energy equals the analytic V (BJ north_star)."""
    pos = np.zeros((2, 4), np.float32)
    pos[0, :3] = [0.5, 0.5, 0.5]
    pos[1, :3] = [0.625, 0.5, 0.5]  # exact fp32 distance 0.125 (sigma = 0.125 below)
    res = orc.lj_rows(pos, [0, 0, 0], [1, 1, 1], [1, 1, 1], rc=0.3, eps=1.0, sigma=0.125)
    assert res["F"][0] == pytest.approx([-24.0 / 0.125, 0, 0], abs=1e-9)
    assert res["F"][1] == pytest.approx([24.0 / 0.125, 0, 0], abs=1e-9)
    assert res["U"].sum() == pytest.approx(0.0, abs=1e-12)
    # analytic two-particle energy at r = 1.5 sigma
    pos[1, 0] = 0.5 + 1.5 * 0.125
    res = orc.lj_rows(pos, [0, 0, 0], [1, 1, 1], [1, 1, 1], rc=0.3, eps=1.0, sigma=0.125)
    V = 4 * ((1 / 1.5) ** 12 - (1 / 1.5) ** 6)
    assert res["U"].sum() == pytest.approx(V, rel=1e-12)
    assert res["F"][0, 0] < 0 < res["F"][1, 0] or res["F"][0, 0] > 0 > res["F"][1, 0]
    # attractive at 1.5 sigma: p (left) is pulled to +x
    assert res["F"][0, 0] > 0


def test_lj_capped_force_closed_form(orc):
    """Reading R22 (cfg5's capped LJ): below r_min = 0.8 sigma the pair force
    has the magnitude of the plain force at r_min, 24 (2/0.8^13 - 1/0.8^7) =
    758.674 (the SURVEY §8(c) value), along the pair axis, and the energy is
    V(r_min); at and above r_min the capped pair is the plain one."""
    f08 = 24.0 * (2.0 / 0.8 ** 13 - 1.0 / 0.8 ** 7)
    assert f08 == pytest.approx(758.67, abs=5e-3)
    pos = np.zeros((2, 4), np.float32)
    pos[0, :3] = [2.0, 2.0, 2.0]
    for d, capped in ((0.5, True), (0.25, True), (0.8125, False), (1.5, False)):
        pos[1, :3] = [2.0, 2.0 + d, 2.0]  # exact fp32 offsets along y
        res = orc.lj_rows(pos, [0, 0, 0], [8, 8, 8], [1, 1, 1], rc=2.5, r_min=0.8)
        plain = orc.lj_rows(pos, [0, 0, 0], [8, 8, 8], [1, 1, 1], rc=2.5)
        if capped:
            assert res["F"][0] == pytest.approx([0.0, -f08, 0.0], rel=1e-12, abs=1e-9)
            assert res["F"][1] == pytest.approx([0.0, f08, 0.0], rel=1e-12, abs=1e-9)
            assert res["U"].sum() == pytest.approx(orc.lj_V(0.8), rel=1e-12)
        else:
            assert np.array_equal(res["F"], plain["F"])
            assert res["U"].sum() == pytest.approx(plain["U"].sum(), rel=1e-15)


def test_lj_cutoff_strict_and_periodic_image(orc):
    """R6 strict inclusion; the minimum image across a periodic face gives the
    same force as the direct pair (PAPER.md:166 periodic BCs)."""
    lo, hi, per = [0, 0, 0], [10, 10, 10], [1, 1, 1]
    pos = np.zeros((2, 4), np.float32)
    pos[0, :3] = [0.25, 5, 5]
    pos[1, :3] = [9.25, 5, 5]  # image distance exactly 1.0
    res = orc.lj_rows(pos, lo, hi, per, rc=2.5)
    assert res["F"][0] == pytest.approx([24.0, 0, 0], rel=1e-12)  # pushed to +x
    pos[1, :3] = [2.75, 5, 5]  # distance exactly 2.5 == rc: excluded (strict)
    res = orc.lj_rows(pos, lo, hi, per, rc=2.5)
    assert res["npair"].sum() == 0 and np.all(res["F"] == 0)
    pos[1, :3] = [np.nextafter(np.float32(2.75), np.float32(0)), 5, 5]
    res = orc.lj_rows(pos, lo, hi, per, rc=2.5)
    assert res["npair"].sum() == 2
    # non-periodic: no image
    res = orc.lj_rows(np.array([[0.25, 5, 5, 0], [9.25, 5, 5, 0]], np.float32), lo, hi,
                      [0, 1, 1], rc=2.5)
    assert res["npair"].sum() == 0


def _sc_lattice_sum(a, rc, eps=1.0, sigma=1.0):
    """U/N = 1/2 sum over SC lattice vectors n != 0 with |n| a < rc of V --
    by integer enumeration (independent of the oracle's pair loop)."""
    m = int(math.ceil(rc / a)) + 1
    u, cnt = 0.0, 0
    for n in itertools.product(range(-m, m + 1), repeat=3):
        if n == (0, 0, 0):
            continue
        r = a * math.sqrt(n[0] ** 2 + n[1] ** 2 + n[2] ** 2)
        if r < rc:
            sr6 = (sigma / r) ** 6
            u += 0.5 * 4 * eps * (sr6 * sr6 - sr6)
            cnt += 1
    return u, cnt


def test_lj_perfect_lattice_closed_form(orc):
    """Exactly representable SC lattice (a = 9/8): F == 0 by symmetry and U/N
    equals the lattice sum; 56 neighbours inside rc = 2.5 at rho = 0.8 spacing."""
    a = 1.125
    s = inputs.lj_lattice_system(16, 16, 16, jitter_key=(0,), a=a, jitter=0.0)
    res = orc.lj_rows(s.pos, s.lo, s.hi, s.periodic, rc=2.5)
    u_ref, cnt = _sc_lattice_sum(a, 2.5)
    assert np.max(np.abs(res["F"])) < 1e-10
    assert np.all(res["npair"] == cnt)
    assert res["U"].mean() == pytest.approx(u_ref, rel=1e-12)
    # rho = 0.8 spacing: neighbour shells |n|^2 <= 5 -> 6 + 12 + 8 + 6 + 24 = 56
    _, cnt08 = _sc_lattice_sum(inputs.A_RHO08, 2.5)
    assert cnt08 == 56


def test_lj_newton_third_law_cfg1(orc):
    """Sum of forces ~ 0 (pairwise antisymmetry) on BJ configs[0]."""
    s = inputs.cfg1()
    res = orc.lj_rows(s.pos, s.lo, s.hi, s.periodic, rc=2.5)
    tot = res["F"].sum(axis=0)
    scale = np.abs(res["F"]).sum()
    assert np.all(np.abs(tot) < 1e-12 * scale)
    rms = np.sqrt(np.mean(res["F"] ** 2))
    assert 5.0 < rms < 20.0  # liquid-like jittered lattice (~10)


# ------------------------------------------------------------------ cells
def test_wrap_rule_adversarial(orc):
    """R1: half-open [lo, hi); -tiny wraps to lo (fl(-tiny + L) == L case)."""
    lo, hi = np.float32(0.0), np.float32(17.235477)
    tiny = np.float32(1e-9)
    xs = np.array([0.0, -tiny, hi, np.nextafter(hi, np.float32(0)), hi + np.float32(1.0),
                   np.float32(-1.0), np.float32(5.0)], np.float32)
    pos = np.zeros((xs.size, 4), np.float32)
    pos[:, 0] = xs
    pos[:, 1] = 1.0
    pos[:, 2] = 1.0
    w, bad = orc.wrap(pos, [lo, 0, 0], [hi, 20, 20], [1, 1, 1])
    assert bad == 0
    x = w[:, 0]
    assert np.all(x >= lo) and np.all(x < hi)
    assert x[0] == 0.0 and x[1] == 0.0 and x[2] == 0.0
    assert x[3] == np.nextafter(hi, np.float32(0))
    assert x[4] == pytest.approx(1.0, abs=1e-5)
    assert x[5] == pytest.approx(float(hi) - 1.0, abs=1e-5)
    # non-periodic out-of-range is reported, not wrapped
    _, bad = orc.wrap(pos, [lo, 0, 0], [hi, 20, 20], [0, 1, 1])
    assert bad == 4


def _check_cell_list(cl, pos_wrapped, lo, hi):
    n = pos_wrapped.shape[0]
    nc = cl["ncell"]
    count, start, perm, cell_of = cl["count"], cl["start"], cl["perm"], cl["cell_of"]
    assert count.sum() == n and start[-1] == n and start[0] == 0
    assert np.all(np.diff(start) == count)
    assert np.array_equal(np.sort(perm), np.arange(n))
    keys = cell_of[perm]
    assert np.all(np.diff(keys) >= 0)
    same = np.diff(keys) == 0
    assert np.all(np.diff(perm)[same] > 0)  # stable: ties in storage order
    # each particle lies in its cell (fp64, up to one fp32 rounding)
    c = np.stack([cell_of % nc[0], (cell_of // nc[0]) % nc[1], cell_of // (nc[0] * nc[1])], 1)
    ext = hi.astype(np.float64) - lo.astype(np.float64)
    w = ext / nc
    x = pos_wrapped[:, :3].astype(np.float64) - lo
    tol = 4e-7 * ext
    assert np.all(x >= c * w - tol) and np.all(x < (c + 1) * w + tol)


def test_cell_list_invariants_cfg1_shuffled(orc):
    s = inputs.shuffled(inputs.cfg1(), (11,))
    cl = orc.cell_list(s.pos, s.lo, s.hi, s.periodic, rv=2.8)
    assert list(cl["ncell"]) == [6, 6, 6]
    _check_cell_list(cl, cl["pos"], s.lo, s.hi)
    assert cl["count"].mean() == pytest.approx(4096 / 216)


def test_cell_list_adversarial_faces(orc):
    """Particles exactly on cell faces, at lo, at hi - ulp, all in one cell."""
    lo = np.zeros(3, np.float32)
    hi = np.full(3, 9.0, np.float32)
    nc, iw = orc.cell_grid(lo, hi, 2.8)
    assert list(nc) == [3, 3, 3]
    faces = np.array([0.0, 3.0, 6.0, np.nextafter(np.float32(9.0), np.float32(0)),
                      np.nextafter(np.float32(3.0), np.float32(0)), 4.5], np.float32)
    pts = np.array(list(itertools.product(faces, repeat=3)), np.float32)
    pos = np.zeros((pts.shape[0] + 50, 4), np.float32)
    pos[:pts.shape[0], :3] = pts
    pos[pts.shape[0]:, :3] = 1.0  # 50 particles in one cell
    cl = orc.cell_list(pos, lo, hi, [1, 1, 1], rv=2.8)
    _check_cell_list(cl, cl["pos"], lo, hi)
    # x = 3.0 exactly: fl(3 * fl(3/9)) rounds to 1.0 -> cell 1
    i = np.where((pts == [3.0, 0.0, 0.0]).all(1))[0][0]
    assert cl["cell_of"][i] == 1
    assert cl["count"].max() >= 50


def test_pair_d2_symmetric_and_periodic(orc):
    """R4: d2(i,j) == d2(j,i) bitwise; across the face equals the direct
    distance of the shifted pair to fp32 accuracy."""
    r = np.random.default_rng(5)
    lo, hi, per = [0, 0, 0], [137.88, 137.88, 68.94], [1, 1, 1]
    for _ in range(2000):
        xi = r.uniform(0, [137.88, 137.88, 68.94]).astype(np.float32)
        xj = (xi + r.uniform(-3, 3, 3)).astype(np.float32)
        xj = np.where(xj >= np.float32(hi), xj - np.float32(hi), xj)
        xj = np.where(xj < 0, xj + np.float32(hi), xj).astype(np.float32)
        d1 = orc.pair_d2(xi, xj, lo, hi, per)
        d2 = orc.pair_d2(xj, xi, lo, hi, per)
        assert d1 == d2
        e = xj.astype(np.float64) - xi.astype(np.float64)
        L = np.asarray(hi, np.float32).astype(np.float64)
        e = np.where(e > L / 2, e - L, np.where(e < -L / 2, e + L, e))
        assert float(d1) == pytest.approx(float((e * e).sum()), rel=1e-5, abs=1e-6)


# ------------------------------------------------------------------ Verlet
def _fp64_pairs(pos, lo, hi, per):
    x = pos[:, :3].astype(np.float64)
    L = (np.asarray(hi, np.float32) - np.asarray(lo, np.float32)).astype(np.float64)
    e = x[None, :, :] - x[:, None, :]
    for d in range(3):
        if per[d]:
            e[..., d] = np.where(e[..., d] > L[d] / 2, e[..., d] - L[d],
                                 np.where(e[..., d] < -L[d] / 2, e[..., d] + L[d], e[..., d]))
    return (e * e).sum(-1)


@pytest.mark.parametrize("per", [(1, 1, 1), (1, 0, 1)])
def test_verlet_brute_force_band(orc, per):
    """R5 against an independent numpy fp64 O(N^2): every pair clearly inside
    r_v is listed, every pair clearly outside is not, sets are symmetric."""
    s = inputs.random_box(1500, 12.0, (7,), periodic=per)
    rv = 2.8
    rp, cols, sh = orc.verlet_rows(s.pos, s.lo, s.hi, s.periodic, rv)
    n = s.n
    d2 = _fp64_pairs(s.pos, s.lo, s.hi, per)
    np.fill_diagonal(d2, np.inf)
    M = np.zeros((n, n), bool)
    for i in range(n):
        M[i, cols[rp[i]:rp[i + 1]]] = True
    rv2 = rv * rv
    assert np.all(M[d2 < rv2 * (1 - 1e-6)])
    assert not np.any(M[d2 > rv2 * (1 + 1e-6)])
    assert np.array_equal(M, M.T)
    # shift codes: only on periodic axes, and consistent with the jump
    if sh.size:
        assert np.all(sh[:, 1] == 0) if per[1] == 0 else True


def test_verlet_cfg1_counts(orc):
    s = inputs.cfg1()
    rows = np.arange(0, s.n, 7)
    rp, cols, _ = orc.verlet_rows(s.pos, s.lo, s.hi, s.periodic, 2.8, rows=rows)
    cnt = np.diff(rp)
    # SC rho = 0.8 lattice + 0.05 jitter: the shells |n|^2 <= 6 lie inside 2.8
    # (6 a^2 = 6.96 < 7.84 < 8 a^2 = 9.28): 6+12+8+6+24+24 = 80 per particle.
    assert np.all(cnt == 80)


# ------------------------------------------------------------------ VV / NVE
def test_vv_energy_conservation_and_momentum(orc):
    """PAPER.md:166 'the total energy was conserved'; reading R25 bound 1e-3
    on the shifted energy; total momentum conserved (pairwise forces)."""
    s = inputs.lj_lattice_system(8, 8, 8, jitter_key=(9,), vel_key=(109,))
    x, v, tr = orc.vv_run(s.pos, s.vel, s.lo, s.hi, s.periodic, rc=2.5, dt=0.005, nsteps=200)
    E = tr[:, 0] + tr[:, 2]
    drift = np.max(np.abs(E - E[0])) / abs(E[0])
    assert drift < 1e-3
    p0 = s.vel[:, :3].astype(np.float64).sum(0)
    assert np.allclose(v.sum(0), p0, atol=1e-9)
    assert np.all(x >= 0) and np.all(x < s.hi.astype(np.float64))
    # KE changes (the lattice melts): integrator actually moves things
    assert abs(tr[-1, 0] - tr[0, 0]) > 1e-3 * tr[0, 0]


def test_vv_second_order(orc):
    """Velocity Verlet is 2nd order: halving dt reduces the energy error ~4x."""
    s = inputs.lj_lattice_system(6, 6, 6, jitter_key=(8,), vel_key=(108,))
    errs = []
    for dt, n in [(0.004, 50), (0.002, 100)]:
        _, _, tr = orc.vv_run(s.pos, s.vel, s.lo, s.hi, s.periodic, rc=2.5, dt=dt, nsteps=n)
        E = tr[:, 0] + tr[:, 2]
        errs.append(np.max(np.abs(E - E[0])))
    assert 2.5 < errs[0] / errs[1] < 6.0


# ------------------------------------------------------------------ SPH
def test_sph_golden_constants():
    rows = {r[0]: float(r[1]) for r in _golden_rows("sph_constants.txt")}
    p = inputs.cfg4(dp=1 / 16.0)  # parameters only depend on dp through h
    assert p.params["gamma"] == rows["gamma"]
    assert p.params["b"] == pytest.approx(rows["b"], rel=1e-12)
    assert p.params["c0"] == pytest.approx(rows["c0"], rel=1e-10)


def test_sph_kernel_normalisation_and_continuity(orc):
    from scipy.integrate import quad
    h = 0.008125
    W0 = float([r for r in _golden_rows("sph_constants.txt") if r[0] == "W0_h0.008125"][0][1])
    assert orc.sph_W(0.0, h) == pytest.approx(W0, rel=1e-6)
    integral = quad(lambda r: 4 * math.pi * r * r * orc.sph_W(r, h), 0, 2 * h, points=[h],
                    epsabs=0, epsrel=1e-12)[0]
    assert integral == pytest.approx(1.0, abs=1e-10)
    for q in (1.0, 2.0):
        a, b = orc.sph_W(q * h * (1 - 1e-9), h), orc.sph_W(q * h * (1 + 1e-9), h)
        assert a == pytest.approx(b, rel=1e-6, abs=1e-3)
    assert orc.sph_W(2.0 * h, h) == 0.0 and orc.sph_W(3 * h, h) == 0.0
    for q in (0.3, 0.9, 1.2, 1.7, 1.99):
        r, e = q * h, 1e-7 * h
        fd = (orc.sph_W(r + e, h) - orc.sph_W(r - e, h)) / (2 * e)
        assert orc.sph_dWdr(r, h) == pytest.approx(fd, rel=1e-6)


def _sph_lattice_density(dp, h, m):
    """rho = m sum over SC lattice vectors (incl. 0) of W -- enumeration."""
    from oracle import oracle as o
    k = int(math.ceil(2 * h / dp)) + 1
    s = 0.0
    for n in itertools.product(range(-k, k + 1), repeat=3):
        s += o.sph_W(dp * math.sqrt(sum(c * c for c in n)), h)
    return m * s


def test_sph_interior_density_and_hydrostatic_balance(orc):
    """Interior fluid particle of a full lattice: rho = lattice sum of m W;
    sum_q grad W = 0 so a = g (Eq. 1, readings R16-R18)."""
    s = inputs.cfg4(dp=1.0 / 16.0)
    p = s.params
    x = s.pos[:, :3].astype(np.float64)
    centre = np.array([0.5, 0.5, 0.25])
    i = int(np.argmin(((x - centre) ** 2).sum(1)))
    assert s.kind[i] == 0
    rho, P = orc.sph_density_rows(s.pos, s.lo, s.hi, s.periodic, p, rows=[i])
    ref = _sph_lattice_density(p["dp"], p["h"], p["mass"])
    assert rho[0] == pytest.approx(ref, rel=1e-12)
    assert rho[0] == pytest.approx(997.2618283038771, rel=1e-9)  # SURVEY §8(c) pin value
    assert P[0] == pytest.approx(p["b"] * ((rho[0] / p["rho0"]) ** 7 - 1), rel=1e-12)
    n = s.n
    rho_all = np.full(n, rho[0])
    P_all = np.full(n, P[0])
    a = orc.sph_accel_rows(s.pos, s.vel, rho_all, P_all, s.kind, s.lo, s.hi, s.periodic, p,
                           rows=[i])
    assert a[0] == pytest.approx(p["g"], abs=1e-9)


def test_sph_two_particle_pressure_repels(orc):
    """Two fluid particles at distance dp, rho = rho0, P = 1000 Pa:
    a_p = -m (2P / rho0^2) W'(dp) (x_p - x_q)/r  (W' by finite difference);
    antisymmetric; positive pressure repels (reading R17)."""
    s = inputs.cfg4(dp=1.0 / 160.0)
    p = dict(s.params)
    p["g"] = (0.0, 0.0, 0.0)
    dp = p["dp"]
    pos = np.array([[0.5, 0.5, 0.25, 0], [0.5 + dp, 0.5, 0.25, 0]], np.float32)
    r = float(np.float64(pos[1, 0]) - np.float64(pos[0, 0]))
    vel = np.zeros_like(pos)
    rho = np.array([1000.0, 1000.0])
    P = np.array([1000.0, 1000.0])
    a = orc.sph_accel_rows(pos, vel, rho, P, np.zeros(2, np.int32), s.lo, s.hi, s.periodic, p)
    e = 1e-9
    dW = (orc.sph_W(r + e, p["h"]) - orc.sph_W(r - e, p["h"])) / (2 * e)
    expect = -p["mass"] * (2000.0 / 1e6) * dW * (-1.0)  # (x_p - x_q)/r = -1 along x
    assert a[0, 0] == pytest.approx(expect, rel=1e-6)
    assert a[0, 0] < 0 < a[1, 0]  # repulsion
    assert a[1] == pytest.approx(-a[0], rel=1e-12)
    assert abs(a[0, 0]) == pytest.approx(34.8196, rel=1e-4)  # SURVEY §8(c) pin value


def test_sph_viscosity_branches(orc):
    """Eq. 5 (reading R20): Pi = 0 for v = 0 and for a
    receding pair; an approaching pair is pushed apart more.  Parity of the
    constants alpha, eta is unpinned by the paper."""
    s = inputs.cfg4(dp=1.0 / 160.0)
    p = dict(s.params)
    p["g"] = (0.0, 0.0, 0.0)
    dp = p["dp"]
    pos = np.array([[0.5, 0.5, 0.25, 0], [0.5 + dp, 0.5, 0.25, 0]], np.float32)
    rho = np.array([1000.0, 1000.0])
    P = np.array([500.0, 500.0])
    kinds = np.zeros(2, np.int32)

    def acc(vx):
        vel = np.zeros_like(pos)
        vel[0, 0], vel[1, 0] = vx, -vx
        return orc.sph_accel_rows(pos, vel, rho, P, kinds, s.lo, s.hi, s.periodic, p)

    a0, a_app, a_rec = acc(0.0), acc(0.5), acc(-0.5)
    assert np.array_equal(a0, a_rec)
    assert a_app[0, 0] < a0[0, 0] < 0  # approaching: extra repulsion of p (to -x)


def test_sph_momentum_conservation_random(orc):
    """sum_p m (a_p - g) = 0 for an all-fluid system: the Eq. 1 pair terms
    (incl. Pi_pq) are antisymmetric."""
    s = inputs.random_box(400, 0.08, (21,), periodic=(1, 1, 1))
    p = dict(inputs.cfg4(dp=1.0 / 160.0).params)
    r = np.random.default_rng(3)
    vel = np.zeros_like(s.pos)
    vel[:, :3] = r.uniform(-0.2, 0.2, (s.n, 3))
    rho, P = orc.sph_density_rows(s.pos, s.lo, s.hi, s.periodic, p)
    a = orc.sph_accel_rows(s.pos, vel, rho, P, np.zeros(s.n, np.int32), s.lo, s.hi,
                           s.periodic, p)
    net = (a - np.asarray(p["g"])).sum(0)
    assert np.all(np.abs(net) < 1e-9 * np.abs(a - np.asarray(p["g"])).sum())


# ------------------------------------------------------------------ WCSPH stepping (NEXT-3)
def _sph_params(h=0.01, c0=44.294):
    return dict(h=h, mass=1e-3, rho0=1000.0, b=c0 * c0 * 1000.0 / 7.0, gamma=7.0, alpha=0.1,
                c0=c0, eta2=0.01 * h * h, g=(0.0, 0.0, -9.81))


def test_sph_run_free_fall_is_exact(orc):
    """An isolated fluid particle: D = 0, a = g.  The Verlet scheme (reading
    R27) integrates constant acceleration exactly, so x(t) = x0 + g t^2 / 2
    and v(t) = g t with t = sum dt; dt (R28) = cfl * min(sqrt(h/|g|), h/c0)."""
    p = _sph_params()
    pos = np.array([[0.5, 0.5, 0.5, 0.0]], np.float32)
    vel = np.zeros((1, 4), np.float32)
    x, v, rho, dt = orc.sph_run(pos, vel, np.array([1000.0]), np.zeros(1, np.int32), [0, 0, 0],
                                [1, 1, 1], [0, 0, 0], p, 120, cfl=0.2, every=40)
    dt_ref = 0.2 * min(math.sqrt(p["h"] / 9.81), p["h"] / p["c0"])
    assert np.allclose(dt, dt_ref, rtol=1e-14)
    t = dt.sum()
    assert x[0, 2] == pytest.approx(0.5 - 0.5 * 9.81 * t * t, abs=1e-14)
    assert v[0, 2] == pytest.approx(-9.81 * t, rel=1e-12)
    assert rho[0] == 1000.0 and x[0, 0] == 0.5 and v[0, 0] == 0.0


def test_sph_run_continuity_sign(orc):
    """Eq. 2 with reading R26: approaching particles compress
    (density rises), receding ones expand; the two densities stay equal."""
    p = dict(_sph_params(), g=(0.0, 0.0, 0.0), alpha=0.0)
    for vx, sign in ((1.0, 1.0), (-1.0, -1.0)):
        pos = np.array([[0.5, 0.5, 0.5, 0], [0.51, 0.5, 0.5, 0]], np.float32)
        vel = np.array([[vx, 0, 0, 0], [-vx, 0, 0, 0]], np.float32)
        _, _, rho, _ = orc.sph_run(pos, vel, np.array([1000.0, 1000.0]), np.zeros(2, np.int32),
                                   [0, 0, 0], [1, 1, 1], [0, 0, 0], p, 3)
        assert sign * (rho[0] - 1000.0) > 0
        assert rho[0] == pytest.approx(rho[1], rel=1e-14)


def test_sph_run_conserves_momentum(orc):
    """No gravity, no boundary particles, periodic box: the pair terms of
    Eq. 1 are antisymmetric, and the leapfrog update v' = v_prev + 2 dt a
    (and the Euler steps) keeps sum m v constant."""
    s = inputs.random_box(300, 0.1, (77,), periodic=(1, 1, 1))
    p = dict(_sph_params(h=0.012), g=(0.0, 0.0, 0.0))
    rng = np.random.default_rng(5)
    vel = np.zeros((s.n, 4), np.float32)
    vel[:, :3] = rng.uniform(-0.5, 0.5, (s.n, 3)).astype(np.float32)
    rho0 = np.full(s.n, 1000.0)
    x, v, rho, dt = orc.sph_run(s.pos, vel, rho0, np.zeros(s.n, np.int32), s.lo, s.hi,
                                s.periodic, p, 25, every=10)
    m0 = vel[:, :3].astype(np.float64).sum(axis=0)
    assert np.max(np.abs(v.sum(axis=0) - m0)) < 1e-11 * np.abs(vel[:, :3]).sum()
    assert np.all(dt > 0) and np.all(np.isfinite(rho))


# ------------------------------------------------------------------ DEM (NEXT-4)
DEM_P = dict(R=0.06, m=1.0, I=1.44e-3, kn=7849.0, kt=2243.0, gn=3.401, gt=0.0, mu=0.5,
             g=(0.0, 0.0, -9.81))


def test_dem_free_fall_leapfrog(orc):
    """Eq. 13 leapfrog without contacts: v_n = n dt g, x_n = x0 + dt^2 g n(n+1)/2."""
    pos = np.array([[0.5, 0.5, 0.5, 0.0]], np.float32)
    z = np.zeros((1, 4), np.float32)
    dt, n = 1e-3, 200
    x, v, w, nh = orc.dem_run(pos, z, z, np.array([0]), [0, 0, 0], [1, 1, 1], [0, 0, 0],
                              [0] * 6, DEM_P, dt, n)
    assert v[0, 2] == pytest.approx(-9.81 * n * dt, rel=1e-12)
    assert x[0, 2] == pytest.approx(0.5 - 9.81 * dt * dt * n * (n + 1) / 2, rel=1e-12)
    assert nh == 0 and np.all(w == 0)


def test_dem_resting_on_floor_closed_form(orc):
    """A damped particle on the z-lo wall settles where the Hertz force
    sqrt(delta/2R) kn delta balances m g: delta* = (m g sqrt(2R)/kn)^(2/3)
    (Eqs. 9, 11); gamma_n raised so the oscillation dies out quickly."""
    p = dict(DEM_P, gn=300.0)
    pos = np.array([[0.5, 0.5, p["R"], 0.0]], np.float32)
    z = np.zeros((1, 4), np.float32)
    x, v, _, _ = orc.dem_run(pos, z, z, np.array([0]), [0, 0, 0], [1, 1, 1], [0, 0, 0],
                             [0, 0, 0, 0, 1, 0], p, 1e-3, 20000)
    ds = (p["m"] * 9.81 * math.sqrt(2 * p["R"]) / p["kn"]) ** (2.0 / 3.0)
    assert x[0, 2] == pytest.approx(p["R"] - ds, rel=1e-6)
    assert abs(v[0, 2]) < 1e-9


def test_dem_elastic_head_on_and_momentum(orc):
    """gamma_n = 0, no gravity: a head-on Hertz collision is elastic (speeds
    come back to v0 up to O(dt)) and conserves momentum exactly (F_qp = -F_pq);
    no tangential motion, no spin."""
    p = dict(DEM_P, gn=0.0, g=(0.0, 0.0, 0.0))
    pos = np.array([[0.4, 0.5, 0.5, 0], [0.6, 0.5, 0.5, 0]], np.float32)
    vel = np.array([[0.5, 0, 0, 0], [-0.5, 0, 0, 0]], np.float32)
    z = np.zeros((2, 4), np.float32)
    x, v, w, nh = orc.dem_run(pos, vel, z, np.array([0, 1]), [0, 0, 0], [1, 1, 1], [0, 0, 0],
                              [0] * 6, p, 2e-5, 20000)
    assert nh == 0  # separated again
    assert v[0, 0] == pytest.approx(-0.5, rel=2e-3) and v[1, 0] == pytest.approx(0.5, rel=2e-3)
    assert abs(v[:, 0].sum()) < 1e-12 and np.all(w == 0)


def test_dem_oblique_friction_momentum_and_spin(orc):
    """An oblique collision with friction (Eqs. 10, 12, Coulomb cap): linear
    momentum is conserved to rounding, both grains get the same torque
    (-R n x F_t for each ordered pair), so they spin equally, and friction
    takes kinetic energy away."""
    p = dict(DEM_P, g=(0.0, 0.0, 0.0))
    pos = np.array([[0.4, 0.5, 0.5, 0], [0.6, 0.53, 0.5, 0]], np.float32)
    vel = np.array([[0.5, 0, 0, 0], [-0.5, 0, 0, 0]], np.float32)
    z = np.zeros((2, 4), np.float32)
    x, v, w, nh = orc.dem_run(pos, vel, z, np.array([0, 1]), [0, 0, 0], [1, 1, 1], [0, 0, 0],
                              [0] * 6, p, 2e-5, 20000)
    assert np.max(np.abs(v.sum(axis=0))) < 1e-12
    assert np.abs(w[0, 2]) > 1e-3 and w[0] == pytest.approx(w[1], rel=1e-9, abs=1e-12)
    ke0, ke1 = 0.5 * 2 * 0.25, 0.5 * np.sum(v * v) + 0.5 * p["I"] * np.sum(w * w)
    assert ke1 < ke0


# ------------------------------------------------------------------ round-2 pins
def _gold_vec(name, key):
    for row in _golden_rows(name):
        if row[0] == key:
            return np.array([float(v) for v in row[1:4]])
    raise KeyError(key)


def test_sph_viscosity_value_hand_computed(orc):
    """Eq. 5 VALUE (not only its branch): Pi_pq and the resulting two-particle
    accelerations of an approaching pair, hand-computed in
    tests/golden/sph_viscosity_pair.txt from PAPER.md:332, 344-350 with the
    R20 constants.  Distinct densities and an oblique, non-axis velocity make a
    dropped h in mu, rho_p in place of rhobar, a dropped eta^2, a flipped
    branch or a transposed v/r fail."""
    h = 0.01
    prm = dict(h=h, mass=1e-3, alpha=0.1, c0=44.29446918449, eta2=0.01 * h * h,
               g=(0.0, 0.0, 0.0))
    pos = np.array([[0.5, 0.5, 0.25, 0], [0.5078125, 0.50390625, 0.25, 0]], np.float32)
    vel = np.array([[0.375, -0.125, 0.25, 0], [-0.25, 0.125, 0.0, 0]], np.float32)
    rho = np.array([1000.0, 1010.0])
    P = np.array([500.0, 1500.0])
    lo, hi, per = [0, 0, 0], [1, 1, 1], [0, 0, 0]
    a = orc.sph_accel_rows(pos, vel, rho, P, np.zeros(2, np.int32), lo, hi, per, prm)
    ap = _gold_vec("sph_viscosity_pair.txt", "a_p")
    assert a[0] == pytest.approx(ap, rel=1e-12, abs=1e-9)
    assert a[1] == pytest.approx(-ap, rel=1e-12, abs=1e-9)  # equal masses: a_q = -a_p
    # the same pair receding (velocities negated): Pi = 0, pressure term only
    a_rec = orc.sph_accel_rows(pos, -vel, rho, P, np.zeros(2, np.int32), lo, hi, per, prm)
    ap0 = _gold_vec("sph_viscosity_pair.txt", "a_p_no_visc")
    assert a_rec[0] == pytest.approx(ap0, rel=1e-12, abs=1e-9)
    # the viscous part alone is -m Pi grad_p W: its ratio to the pressure part
    # is Pi / ((P_p + P_q)/(rho_p rho_q)) (hand value of Pi)
    Pi = _gold_vec("sph_viscosity_pair.txt", "Pi")[0]
    assert (a[0, 0] - a_rec[0, 0]) / a_rec[0, 0] == pytest.approx(Pi / (2000.0 / 1.01e6),
                                                                    rel=1e-10)


def test_lj_virial_pair_closed_form(orc):
    """Virial W = 1/2 sum_i sum_j (x_i - x_j) . F_ij of
    one pair at r = 1.5 sigma equals r F(r) = -1.7370432465692334 (hand value,
    tests/golden/sph_viscosity_pair.txt); a wrong sign or a missing 1/2 fails."""
    pos = np.zeros((2, 4), np.float32)
    pos[0, :3] = [2.0, 3.0, 3.0]
    pos[1, :3] = [3.5, 3.0, 3.0]
    res = orc.lj_rows(pos, [0, 0, 0], [8, 8, 8], [1, 1, 1], rc=2.5)
    W = _gold_vec("sph_viscosity_pair.txt", "lj_virial_r1.5")[0]
    assert res["W"].sum() == pytest.approx(W, rel=1e-12)
    assert res["W"][0] == pytest.approx(W / 2, rel=1e-12)


def test_lj_virial_is_minus_scaling_derivative(orc):
    """Thermodynamic identity, independent of the oracle's virial code: for a
    uniform dilation x -> lambda x of positions and box, the shifted energy
    U_s (pairs crossing r_c add V(r_c) - V(r_c) = 0, so U_s is continuous)
    satisfies dU_s/dlambda = sum_pairs r dV/dr = -W at lambda = 1."""
    s = inputs.lj_lattice_system(10, 10, 10, jitter_key=(31,))
    x64 = s.pos[:, :3].astype(np.float64)
    hi64 = s.hi.astype(np.float64)
    vrc = orc.lj_V(2.5)

    def Us(lam):
        p = np.zeros_like(s.pos)
        p[:, :3] = (x64 * lam).astype(np.float32)
        hi = (hi64 * lam).astype(np.float32)
        r = orc.lj_rows(p, [0, 0, 0], hi, [1, 1, 1], rc=2.5)
        return r["U"].sum() - 0.5 * r["npair"].sum() * vrc, r["W"].sum()

    eps = 2e-4
    up, _ = Us(1 + eps)
    um, _ = Us(1 - eps)
    _, W = Us(1.0)
    dU = (up - um) / (2 * eps)
    assert W == pytest.approx(-dU, rel=2e-4)
    assert abs(W) > 100.0  # a non-trivial virial (jittered dense liquid)


@pytest.mark.parametrize("per", [(1, 1, 1), (1, 0, 1)])
def test_verlet_shift_reconstructs_minimum_image(orc, per):
    """Image-shift codes of the Verlet sets: for every
    listed pair x_j + shift L - x_i is the fp64 minimum-image difference (a
    flipped sign is off by 2L), |.| < r_v, and shift = 0 on open axes.  The
    particles sit in slabs next to the faces so most pairs cross one."""
    r = np.random.default_rng(77)
    L = 9.0
    n = 900
    x = r.uniform(0, L, (n, 3))
    face = r.integers(0, 2, (n, 3)).astype(bool)
    x = np.where(face, r.uniform(0, 1.4, (n, 3)), L - r.uniform(1e-3, 1.4, (n, 3)))
    pos = np.zeros((n, 4), np.float32)
    pos[:, :3] = x.astype(np.float32)
    lo, hi = np.zeros(3, np.float32), np.full(3, L, np.float32)
    rv = 2.8
    rp, cols, sh = orc.verlet_rows(pos, lo, hi, np.asarray(per, np.int32), rv)
    rows = np.repeat(np.arange(n), np.diff(rp))
    xi = pos[rows, :3].astype(np.float64)
    xj = pos[cols, :3].astype(np.float64)
    Lv = hi.astype(np.float64) - lo.astype(np.float64)
    rec = xj + sh.astype(np.float64) * Lv - xi
    e = xj - xi
    for d in range(3):
        if per[d]:
            e[:, d] = np.where(e[:, d] > Lv[d] / 2, e[:, d] - Lv[d],
                               np.where(e[:, d] < -Lv[d] / 2, e[:, d] + Lv[d], e[:, d]))
        else:
            assert np.all(sh[:, d] == 0)
    assert np.max(np.abs(rec - e)) < 1e-5
    assert np.all(np.sqrt((rec * rec).sum(1)) < rv * (1 + 1e-6))
    assert np.count_nonzero(sh) > 0.3 * sh.shape[0]  # the case is face-dominated


def test_md_cells_run_matches_brute_force_trajectory(orc):
    """The CPU cell-list + Verlet + VV baseline reorganises the
    O(N^2) sum exactly: same trajectory as orc_vv_run (brute force) up to
    summation order over 60 steps with several list rebuilds, and the same
    number of pairs inside r_c at every step."""
    s = inputs.lj_lattice_system(12, 12, 12, jitter_key=(41,), vel_key=(141,))
    x0, v0, tr0 = orc.vv_run(s.pos, s.vel, s.lo, s.hi, s.periodic, rc=2.5, dt=0.005, nsteps=60)
    x1, v1, tr1, nb = orc.md_cells_run(s.pos, s.vel, s.lo, s.hi, s.periodic, rc=2.5, skin=0.3,
                                       dt=0.005, nsteps=60)
    assert nb >= 3  # rebuilds happened (rebuild at skin/2)
    assert np.array_equal(tr0[:, 3], tr1[:, 3])
    assert np.max(np.abs(x1 - x0)) < 1e-9
    assert np.max(np.abs(v1 - v0)) < 1e-8
    assert np.allclose(tr1[:, :3], tr0[:, :3], rtol=1e-10, atol=1e-9)
