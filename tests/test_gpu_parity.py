"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Integer structures (cell ids, counts, starts, permutation, neighbour sets,
pair counts) must be bit-exact; forces / densities / accelerations within the
BASELINE.json north_star bar: max per-component |err| / RMS(ref) <= 1e-4.
"""
import numpy as np
import pytest

from paper_1804_07598_b200 import inputs

pytestmark = pytest.mark.gpu

TOL = 1e-4  # BJ north_star: forces and densities within 1e-4 of the RMS


@pytest.fixture(scope="module")
def pm():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1804_07598_b200 import build, pm as pmmod
    build.build()
    pmmod.lib()
    return pmmod


def f32(x):
    return np.float32(x)


def rv32(rc, skin):
    return np.float32(np.float32(rc) + np.float32(skin))  # reading R5


def make_ctx(pm, s, rc=2.5, skin=0.3, r_min=0.0, **kw):
    c = pm.Context(**kw)
    c.set_domain(s.lo, s.hi, s.periodic)
    c.set_cutoff(rc, skin)
    c.set_lj(1.0, 1.0, 1.0, r_min)
    c.place(s.pos, s.vel, s.gid, s.kind)
    return c


def idx_of_gid(s):
    inv = np.empty(int(s.gid.max()) + 1, np.int64)
    inv[s.gid] = np.arange(s.n)
    return inv


# ---------------------------------------------------------------- cells
@pytest.mark.parametrize("name", ["cfg1_shuffled", "cfg2", "faces_bigcell", "sparse_thin"])
def test_cells_bit_exact(pm, orc, name):
    if name == "cfg1_shuffled":
        s = inputs.shuffled(inputs.cfg1(), (11,))
    elif name == "sparse_thin":  # < 4 particles per cell: lane-per-cell sort (k_segsort_thin)
        s = inputs.random_box(6000, 40.0, (17,))
        r = np.random.default_rng(5)  # a few crowded cells take the warp path inside it
        pts = r.uniform(10.0, 12.7, (60, 3)).astype(np.float32)
        s.pos[:60, :3] = pts
    elif name == "cfg2":
        s = inputs.cfg2()
    else:
        import itertools
        faces = np.array([0.0, 3.0, 6.0, np.nextafter(f32(9.0), f32(0)),
                          np.nextafter(f32(3.0), f32(0)), 4.5, -1e-9, 9.0], np.float32)
        pts = np.array(list(itertools.product(faces, repeat=3)), np.float32)
        r = np.random.default_rng(0)
        big = r.uniform(0.1, 2.9, (3000, 3)).astype(np.float32)  # one 3000-particle cell
        mid = r.uniform(3.0, 6.0, (40, 3)).astype(np.float32)  # a 40-particle cell
        xyz = np.concatenate([pts, big, mid])
        perm = r.permutation(xyz.shape[0])
        pos = np.zeros((xyz.shape[0], 4), np.float32)
        pos[:, :3] = xyz[perm]
        s = inputs.System(pos=pos, vel=np.zeros_like(pos), gid=np.arange(pos.shape[0]),
                          lo=np.zeros(3, np.float32), hi=np.full(3, 9.0, np.float32),
                          periodic=np.ones(3, np.int32))
    c = make_ctx(pm, s)
    c.build_cells()
    g = c.get_cells()
    ref = orc.cell_list(s.pos, s.lo, s.hi, s.periodic, rv=rv32(2.5, 0.3))
    assert np.array_equal(g["cell_of"], ref["cell_of"])
    assert np.array_equal(g["start"], ref["start"])
    assert np.array_equal(g["perm"], ref["perm"])
    # the particle arrays were reordered into cell order
    st = c.get_state()
    assert np.array_equal(st["gid"], s.gid[ref["perm"]])
    assert np.array_equal(st["pos"], ref["pos"][ref["perm"]])
    c.close()


# ---------------------------------------------------------------- Verlet
def _row_sets_equal(rp, col, gids, ref_rp, ref_cols, ref_gid_of_col):
    for r in range(len(gids)):
        got = np.sort(col[rp[r]:rp[r + 1]])
        exp = np.sort(ref_gid_of_col[ref_cols[ref_rp[r]:ref_rp[r + 1]]])
        if not np.array_equal(got, exp):
            return r
    return -1


@pytest.mark.parametrize("name", ["cfg1", "random_mixed_bc", "cfg2_sampled"])
def test_verlet_sets_bit_exact(pm, orc, name):
    if name == "cfg1":
        s = inputs.shuffled(inputs.cfg1(), (12,))
    elif name == "random_mixed_bc":
        s = inputs.random_box(3000, 14.0, (13,), periodic=(1, 0, 1))
    else:
        s = inputs.cfg2()
    c = make_ctx(pm, s)
    c.build_verlet()
    rp, col = c.get_verlet()
    st = c.get_state()
    gid_rows = st["gid"]
    inv = idx_of_gid(s)
    if name == "cfg2_sampled":
        pick = np.random.default_rng(1).choice(s.n, 200, replace=False)
    else:
        pick = np.arange(s.n)
    rows_storage = inv[gid_rows[pick]]
    rrp, rcols, _ = orc.verlet_rows(s.pos, s.lo, s.hi, s.periodic, rv32(2.5, 0.3),
                                    rows=rows_storage, want_shift=False)
    sub_rp = np.concatenate([[0], np.cumsum(rp[pick + 1] - rp[pick])])
    sub_col = np.concatenate([col[rp[i]:rp[i + 1]] for i in pick]) if len(pick) else col[:0]
    bad = _row_sets_equal(sub_rp, sub_col, gid_rows[pick], rrp, rcols, s.gid)
    assert bad < 0, f"row {bad} (gid {gid_rows[pick][bad]}) differs"
    assert c.count()["nnz"] == rp[-1]
    c.close()


@pytest.mark.parametrize("L,n,per", [(8.5, 600, (1, 1, 1)), (11.5, 1500, (1, 1, 1)),
                                     (14.5, 2500, (1, 0, 1)), (25.0, 300, (1, 1, 1)),
                                     (9.0, 700, (0, 1, 1)), (40.0, 3000, (1, 1, 0))])
def test_verlet_small_grids_and_sparse(pm, orc, L, n, per):
    """3, 4 and 5 cells per periodic axis (every stencil wraps), sparse boxes
    (a warp spans many cells: whole-row path), mixed boundary conditions."""
    s = inputs.random_box(n, L, (31, n), periodic=per)
    c = make_ctx(pm, s)
    c.build_verlet()
    rp, col = c.get_verlet()
    st = c.get_state()
    inv = idx_of_gid(s)
    rrp, rcols, _ = orc.verlet_rows(s.pos, s.lo, s.hi, s.periodic, rv32(2.5, 0.3),
                                    rows=inv[st["gid"]], want_shift=False)
    bad = _row_sets_equal(rp, col, st["gid"], rrp, rcols, s.gid)
    assert bad < 0, f"row {bad} differs"
    c.close()


@pytest.mark.parametrize("per", [(1, 1, 1), (1, 0, 1)])
def test_cell_div2_cells_lists_forces(pm, orc, per):
    """Reading R2's second grid (pm_opts.cell_div = 2: cells of side >= r_v/2,
    5 x 5 x 5 stencil): cell ids / starts / perm bit-exact against the
    oracle's cell_div = 2 grid, the same Verlet sets as the brute-force
    oracle, forces within the bar, and a short run that follows the
    cell_div = 1 one."""
    s = inputs.random_box(3000, 15.0, (19,), periodic=per)
    s2 = inputs.lj_lattice_system(14, 14, 14, jitter_key=(18,), vel_key=(118,))
    c = make_ctx(pm, s, r_min=0.8, cell_div=2)
    c.build_cells()
    g = c.get_cells()
    ref = orc.cell_list(s.pos, s.lo, s.hi, s.periodic, rv=rv32(2.5, 0.3), cell_div=2)
    assert np.array_equal(g["cell_of"], ref["cell_of"])
    assert np.array_equal(g["start"], ref["start"])
    assert np.array_equal(g["perm"], ref["perm"])
    c.build_verlet()
    rp, col = c.get_verlet()
    st = c.get_state()
    rrp, rcols, _ = orc.verlet_rows(s.pos, s.lo, s.hi, s.periodic, rv32(2.5, 0.3),
                                    rows=idx_of_gid(s)[st["gid"]], want_shift=False)
    bad = _row_sets_equal(rp, col, st["gid"], rrp, rcols, s.gid)
    assert bad < 0, f"row {bad} differs"
    c.compute_lj()
    st = c.get_state()
    fr = orc.lj_rows(s.pos, s.lo, s.hi, s.periodic, rc=2.5, r_min=0.8,
                     rows=idx_of_gid(s)[st["gid"]])
    assert orc.normalized_max_err(st["force"][:, :3].astype(np.float64), fr["F"]) <= TOL
    c.close()
    out = []
    for cd in (1, 2):
        c = make_ctx(pm, s2, cell_div=cd)
        r = c.step_vv(0.005, 20)
        out.append((pm.sorted_by_gid(c.get_state()), r["rebuilds"]))
        c.close()
    assert out[0][1] == out[1][1]
    assert np.max(np.abs(out[0][0]["pos"][:, :3] - out[1][0]["pos"][:, :3])) < 1e-4


@pytest.mark.parametrize("L,n,per", [(8.5, 600, (1, 1, 1)), (14.5, 2500, (1, 0, 1))])
def test_verlet_sets_with_image_shifts(pm, orc, L, n, per):
    """R5 compares lists as sets of (gid_i, gid_j, image shift): with 3-5
    cells per periodic axis every stencil wraps; the shifts of
    pm_get_verlet_shifts equal the oracle's, entry for entry."""
    s = inputs.random_box(n, L, (33, n), periodic=per)
    c = make_ctx(pm, s)
    c.build_verlet()
    rp, col = c.get_verlet()
    sh = c.get_verlet_shifts()
    st = c.get_state()
    inv = idx_of_gid(s)
    rrp, rcols, rsh = orc.verlet_rows(s.pos, s.lo, s.hi, s.periodic, rv32(2.5, 0.3),
                                      rows=inv[st["gid"]], want_shift=True)
    nonzero = 0
    for r in range(s.n):
        got = sorted(zip(col[rp[r]:rp[r + 1]].tolist(), map(tuple, sh[rp[r]:rp[r + 1]].tolist())))
        exp = sorted(zip(s.gid[rcols[rrp[r]:rrp[r + 1]]].tolist(),
                         map(tuple, rsh[rrp[r]:rrp[r + 1]].tolist())))
        assert got == exp, f"row {r}"
        nonzero += sum(1 for _, t in got if any(t))
    assert nonzero > 0  # some pairs cross a periodic face
    c.close()


def test_verlet_capacity_overflow_retry(pm, orc):
    """A tiny initial capacity overflows; the library grows it and retries."""
    s = inputs.cfg1()
    c = make_ctx(pm, s, nbr_cap=8)
    c.build_verlet()
    rp, col = c.get_verlet()
    assert np.all(np.diff(rp) == 80)  # SC rho=0.8 + jitter: 80 inside 2.8 (pinned)
    c.close()


# ---------------------------------------------------------------- LJ forces
@pytest.mark.parametrize("name", ["cfg1", "cfg2_sampled", "random_mixed_bc"])
def test_lj_forces_parity(pm, orc, name):
    if name == "cfg1":
        s = inputs.shuffled(inputs.cfg1(), (14,))
        pick = None
    elif name == "cfg2_sampled":
        s = inputs.cfg2()
        pick = np.random.default_rng(2).choice(s.n, 512, replace=False)
    else:
        s = inputs.lj_lattice_system(14, 14, 14, jitter_key=(15,), jitter=0.12)
        s.periodic = np.array([1, 1, 0], np.int32)
        s.hi[2] = s.hi[2] + np.float32(0.5)
        pick = None
    c = make_ctx(pm, s)
    c.build_verlet()
    c.compute_lj(want_energy=True)
    st = c.get_state()
    th = c.thermo(recompute=False)
    inv = idx_of_gid(s)
    rows = np.arange(s.n) if pick is None else pick
    rows_storage = inv[st["gid"][rows]]
    ref = orc.lj_rows(s.pos, s.lo, s.hi, s.periodic, rc=2.5, rows=rows_storage)
    F = st["force"][rows, :3].astype(np.float64)
    err = orc.normalized_max_err(F, ref["F"])
    assert err <= TOL, err
    if pick is None:
        # integer pair count bit-exact; energy/virial to fp32-sum accuracy
        assert th["npairs"] == int(ref["npair"].sum())
        assert th["pe_raw"] == pytest.approx(ref["U"].sum(), rel=1e-5)
        assert th["virial"] == pytest.approx(ref["W"].sum(), rel=1e-5)
        net = F.sum(0)
        assert np.all(np.abs(net) < 1e-4 * np.abs(F).sum())  # Newton (fp32 sums)
    c.close()


@pytest.mark.parametrize("name", ["cfg1", "cfg2_sampled", "random_mixed_bc"])
def test_newton_half_lists_and_forces(pm, orc, name):
    """NEXT-1 half (Newton) lists (pm_set_newton): every row is exactly the
    oracle's full row restricted to partners later in the current (cell)
    order, so each unordered pair appears once; the reduction sweep gives the
    oracle's forces within the north_star bar, and the whole-system pair
    count, energy and virial."""
    if name == "cfg1":
        s = inputs.shuffled(inputs.cfg1(), (14,))
        pick = None
    elif name == "cfg2_sampled":
        s = inputs.cfg2()
        pick = np.random.default_rng(3).choice(s.n, 400, replace=False)
    else:
        s = inputs.lj_lattice_system(14, 14, 14, jitter_key=(15,), jitter=0.12)
        s.periodic = np.array([1, 1, 0], np.int32)
        s.hi[2] = s.hi[2] + np.float32(0.5)
        pick = None
    c = pm.Context()
    c.set_newton(True)
    c.set_domain(s.lo, s.hi, s.periodic)
    c.set_cutoff(2.5, 0.3)
    c.set_lj(1.0, 1.0, 1.0, 0.0)
    c.place(s.pos, s.vel, s.gid, s.kind)
    c.build_verlet()
    rp, col = c.get_verlet()
    st = c.get_state()
    cur_of_gid = np.empty(int(s.gid.max()) + 1, np.int64)
    cur_of_gid[st["gid"]] = np.arange(s.n)
    inv = idx_of_gid(s)
    rows = np.arange(s.n) if pick is None else pick
    rrp, rcols, _ = orc.verlet_rows(s.pos, s.lo, s.hi, s.periodic, rv32(2.5, 0.3),
                                    rows=inv[st["gid"][rows]], want_shift=False)
    for t, i in enumerate(rows):
        full = s.gid[rcols[rrp[t]:rrp[t + 1]]]
        half = np.sort(full[cur_of_gid[full] > i])
        assert np.array_equal(np.sort(col[rp[i]:rp[i + 1]]), half), f"row {i}"
    if pick is None:
        assert rp[-1] * 2 == len(rcols)  # each unordered pair once
    c.compute_lj(want_energy=True)
    st = c.get_state()
    th = c.thermo(recompute=False)
    ref = orc.lj_rows(s.pos, s.lo, s.hi, s.periodic, rc=2.5, rows=inv[st["gid"][rows]])
    err = orc.normalized_max_err(st["force"][rows, :3].astype(np.float64), ref["F"])
    assert err <= TOL, err
    if pick is None:
        assert th["npairs"] == int(ref["npair"].sum())
        assert th["pe_raw"] == pytest.approx(ref["U"].sum(), rel=1e-5)
        assert th["virial"] == pytest.approx(ref["W"].sum(), rel=1e-5)
    c.close()


def test_newton_nve_matches_full_list(pm):
    """The Newton path through pm_step_vv (clear F -> half sweep with
    reductions -> velocity-Verlet kernel, in the CUDA graph with the
    conditional rebuild) follows the full-list trajectory over 30 steps with
    rebuilds (differences: fp32 summation order only); SPH, DEM and
    decomposition refuse half lists."""
    s = inputs.lj_lattice_system(24, 24, 24, jitter_key=(16,), vel_key=(116,))
    out = {}
    for newton in (False, True):
        c = pm.Context()
        c.set_newton(newton)
        c.set_domain(s.lo, s.hi, s.periodic)
        c.set_cutoff(2.5, 0.3)
        c.set_lj(1.0, 1.0, 1.0, 0.0)
        c.place(s.pos, s.vel, s.gid, s.kind)
        r = c.step_vv(0.005, 30)
        out[newton] = (pm.sorted_by_gid(c.get_state()), r["rebuilds"])
        if newton:
            with pytest.raises(pm.PMError) as e:
                c.sph_density()
            assert e.value.code == -2
        c.close()
    a, b = out[False][0], out[True][0]
    assert out[False][1] == out[True][1] and out[True][1] >= 2
    assert np.max(np.abs(a["pos"][:, :3] - b["pos"][:, :3])) < 1e-4
    assert np.max(np.abs(a["vel"][:, :3] - b["vel"][:, :3])) < 1e-3


def test_lj_perfect_lattice_closed_form(pm):
    """Exactly representable SC lattice: F = 0 and U/N = lattice sum (pinned in
    tests/test_oracle_pins.py by integer enumeration)."""
    from test_oracle_pins import _sc_lattice_sum
    s = inputs.lj_lattice_system(16, 16, 16, jitter_key=(0,), a=1.125, jitter=0.0)
    c = make_ctx(pm, s)
    c.build_verlet()
    c.compute_lj(want_energy=True)
    st = c.get_state()
    u_ref, cnt = _sc_lattice_sum(1.125, 2.5)
    assert np.max(np.abs(st["force"][:, :3])) < 1e-4
    th = c.thermo(recompute=False)
    assert th["npairs"] == cnt * s.n
    assert th["pe_raw"] / s.n == pytest.approx(u_ref, rel=1e-6)
    c.close()


def test_forces_bitwise_deterministic(pm):
    s = inputs.cfg1()
    out = []
    for _ in range(2):
        c = make_ctx(pm, s)
        c.build_verlet()
        c.compute_lj()
        out.append(pm.sorted_by_gid(c.get_state())["force"])
        c.close()
    assert np.array_equal(out[0], out[1])


def test_capped_lj_parity(pm, orc):
    """Reading R22 capped force (cfg5 physics) on a dense random cloud."""
    s = inputs.random_box(4000, 12.0, (16,))
    c = make_ctx(pm, s, r_min=0.8)
    c.build_verlet()
    c.compute_lj()
    st = c.get_state()
    inv = idx_of_gid(s)
    ref = orc.lj_rows(s.pos, s.lo, s.hi, s.periodic, rc=2.5, r_min=0.8,
                      rows=inv[st["gid"]])
    assert orc.normalized_max_err(st["force"][:, :3], ref["F"]) <= TOL
    c.close()


# ---------------------------------------------------------------- clustered (cfg5)
@pytest.fixture(scope="module")
def clustered():
    """BJ configs[4] at its full local density: 4 of the 64 Gaussian clusters
    (131,072 particles each, sigma_c = 4, mean density 0.5): cells of ~3000
    particles (block-level sort), rows of up to ~12k entries (per-slice list
    widths), capped LJ (reading R22)."""
    return inputs.cfg5(n_clusters=4)


def test_clustered_cells_lists_forces(pm, orc, clustered):
    s = clustered
    c = make_ctx(pm, s, r_min=0.8)
    c.build_cells()
    g = c.get_cells()
    ref = orc.cell_list(s.pos, s.lo, s.hi, s.periodic, rv=rv32(2.5, 0.3))
    assert ref["count"].max() > 1000  # big cells exercised
    assert np.array_equal(g["cell_of"], ref["cell_of"])
    assert np.array_equal(g["start"], ref["start"])
    assert np.array_equal(g["perm"], ref["perm"])
    c.build_verlet()
    c.compute_lj()
    rp, col = c.get_verlet()
    st = c.get_state()
    lens = np.diff(rp)
    assert lens.max() > 4000 and lens.min() < 50  # strongly non-uniform rows
    # sample rows across the whole length distribution (dense cores included)
    order = np.argsort(lens)
    pick = order[np.linspace(0, len(order) - 1, 48).astype(int)]
    inv = idx_of_gid(s)
    rows_storage = inv[st["gid"][pick]]
    rrp, rcols, _ = orc.verlet_rows(s.pos, s.lo, s.hi, s.periodic, rv32(2.5, 0.3),
                                    rows=rows_storage, want_shift=False)
    sub_rp = np.concatenate([[0], np.cumsum(rp[pick + 1] - rp[pick])])
    sub_col = np.concatenate([col[rp[i]:rp[i + 1]] for i in pick])
    bad = _row_sets_equal(sub_rp, sub_col, st["gid"][pick], rrp, rcols, s.gid)
    assert bad < 0, f"row {bad} differs"
    fr = orc.lj_rows(s.pos, s.lo, s.hi, s.periodic, rc=2.5, r_min=0.8, rows=rows_storage)
    assert orc.normalized_max_err(st["force"][pick, :3], fr["F"]) <= TOL
    c.close()


def test_clustered_row_major_equals_sell(pm, clustered, monkeypatch):
    """Long rows (widest slice >= 512 entries) are stored row-major (each row
    contiguous: whole-sector appends in the build); the entries and their
    order are those of the SELL-32 layout, so a short capped run with rebuilds
    is bitwise the same trajectory either way (PM_ROW_MAJOR=0 forces SELL)."""
    s = clustered
    out = []
    for rm in ("1", "0"):
        monkeypatch.setenv("PM_ROW_MAJOR", rm)
        c = make_ctx(pm, s, r_min=0.8)
        c.set_vlimit(0.15 / 0.005)
        r = c.step_vv(0.005, 4)
        assert r["rebuilds"] >= 2
        st = pm.sorted_by_gid(c.get_state())
        rp, col = c.get_verlet()
        out.append((st, np.diff(rp)))
        c.close()
    (a, la), (b, lb) = out
    assert la.max() > 4000 and np.array_equal(np.sort(la), np.sort(lb))
    assert np.array_equal(a["pos"], b["pos"]) and np.array_equal(a["vel"], b["vel"])


def test_row_major_switches_with_half_lists(pm, clustered):
    """The list layout follows the context: long LJ rows are row-major, half
    (Newton) lists are SELL-32 only, so pm_set_newton switches the layout
    (list and graphs dropped, the next build writes the other kind).  Forces
    full (row-major) -> half (SELL) -> full again: the half-list forces agree
    within the parity tolerance, the two full-list passes bit for bit."""
    s = clustered
    c = make_ctx(pm, s, r_min=0.8)
    c.build_verlet()
    c.compute_lj()
    f1 = pm.sorted_by_gid(c.get_state())["force"][:, :3].astype(np.float64)
    c.set_newton(True)
    c.build_verlet()
    c.compute_lj()
    f2 = pm.sorted_by_gid(c.get_state())["force"][:, :3].astype(np.float64)
    c.set_newton(False)
    c.build_verlet()
    c.compute_lj()
    f3 = pm.sorted_by_gid(c.get_state())["force"][:, :3].astype(np.float64)
    rms = np.sqrt(np.mean(f1 ** 2))
    assert np.max(np.abs(f2 - f1)) / rms <= TOL
    assert np.array_equal(f1, f3)
    c.close()


def test_clustered_short_run_with_vlimit(pm, clustered):
    """Reading R22 dynamics: capped LJ + velocity limit (skin/2)/dt; runs with a
    rebuild (incl. relayout of the list widths) nearly every step."""
    s = clustered
    c = make_ctx(pm, s, r_min=0.8)
    c.set_vlimit(0.15 / 0.005)
    r = c.step_vv(0.005, 6)
    assert r["steps"] == 6 and r["rebuilds"] >= 3
    st = c.get_state()
    assert np.all(np.isfinite(st["pos"])) and np.all(np.isfinite(st["vel"]))
    v = np.linalg.norm(st["vel"][:, :3], axis=1)
    assert v.max() <= 30.0 * (1 + 1e-5)
    assert np.array_equal(np.sort(st["gid"]), np.sort(s.gid))
    c.close()


# ---------------------------------------------------------------- VV / NVE
def test_vv_short_trajectory_vs_oracle(pm, orc):
    """Positions after 50 fp32 steps within 1e-3 sigma of the fp64 oracle
    (SURVEY §8(c) NVE pin; chaos limits longer horizons)."""
    s = inputs.lj_lattice_system(12, 12, 12, jitter_key=(17,), vel_key=(117,))
    c = make_ctx(pm, s)
    stats = c.step_vv(0.005, 50)
    assert stats["steps"] == 50 and stats["rebuilds"] >= 2
    st = pm.sorted_by_gid(c.get_state())
    x, v, tr = orc.vv_run(s.pos, s.vel, s.lo, s.hi, s.periodic, rc=2.5, dt=0.005, nsteps=50)
    L = s.hi.astype(np.float64)
    d = st["pos"][:, :3].astype(np.float64) - x
    d -= L * np.round(d / L)
    assert np.max(np.abs(d)) < 1e-3
    assert np.max(np.abs(st["vel"][:, :3] - v)) < 1e-2
    ke = 0.5 * np.sum(st["vel"][:, :3].astype(np.float64) ** 2)
    assert ke == pytest.approx(tr[-1, 0], rel=1e-3)
    c.close()


def test_nve_energy_drift_cfg2(pm):
    """BJ configs[1]: 1000 NVE steps, rebuild at skin/2; shifted-energy drift
    <= 1e-3 (reading R25; PAPER.md:166 'the total energy was conserved');
    total momentum conserved."""
    s = inputs.cfg2()
    c = make_ctx(pm, s)
    c.build_verlet()
    th0 = c.thermo()
    E0 = th0["ke"] + th0["pe_shift"]
    p0 = s.vel[:, :3].astype(np.float64).sum(0)
    drift = 0.0
    reb = 0
    for _ in range(10):
        r = c.step_vv(0.005, 100)
        reb += r["rebuilds"]
        th = c.thermo()
        drift = max(drift, abs(th["ke"] + th["pe_shift"] - E0) / abs(E0))
    assert drift < 1e-3, drift
    assert 60 <= reb <= 400
    st = c.get_state()
    p = st["vel"][:, :3].astype(np.float64).sum(0)
    assert np.all(np.abs(p - p0) < 1e-2)
    c.close()


def test_step_vv_graph_equals_nongraph(pm):
    """The CUDA-graph step loop (conditional rebuild node) and the plain launch
    loop give bitwise identical trajectories."""
    s = inputs.lj_lattice_system(12, 12, 12, jitter_key=(18,), vel_key=(118,))
    res = []
    for g in (True, False):
        c = make_ctx(pm, s, use_graphs=g)
        r = c.step_vv(0.005, 40)
        res.append((r["rebuilds"], pm.sorted_by_gid(c.get_state())))
        c.close()
    assert res[0][0] == res[1][0]
    for k in ("pos", "vel", "force"):
        assert np.array_equal(res[0][1][k], res[1][1][k])


# ---------------------------------------------------------------- SPH
def _sph_ctx(pm, s):
    p = s.params
    c = pm.Context()
    c.set_domain(s.lo, s.hi, s.periodic)
    c.set_cutoff(2.0 * p["h"], 0.0)
    c.set_sph(p)
    c.place(s.pos, s.vel, s.gid, s.kind)
    c.build_verlet()
    c.sph_density()
    c.sph_forces()
    return c


def test_sph_parity_small_dam(pm, orc):
    """cfg4 geometry at dp = 1/32 with random velocities (exercises Eq. 5):
    densities of all particles and accelerations (a - g) of sampled ones."""
    s = inputs.cfg4(dp=1.0 / 32.0, vel_key=(104,))
    p = s.params
    c = _sph_ctx(pm, s)
    st = c.get_state()
    inv = idx_of_gid(s)
    rho_ref, P_ref = orc.sph_density_rows(s.pos, s.lo, s.hi, s.periodic, p)
    got_rho = st["rho"][np.argsort(st["gid"])]
    assert orc.normalized_max_err(got_rho, rho_ref) <= TOL
    rows = np.random.default_rng(4).choice(s.n, 4000, replace=False)
    a_ref = orc.sph_accel_rows(s.pos, s.vel, rho_ref, P_ref, s.kind, s.lo, s.hi, s.periodic, p,
                               rows=rows)
    pos_of_gid = np.argsort(st["gid"])
    a_got = st["force"][pos_of_gid[s.gid[rows]], :3].astype(np.float64)
    g = np.asarray(p["g"])
    fluid = s.kind[rows] == 0
    assert orc.normalized_max_err(a_got[fluid] - g, a_ref[fluid] - g) <= TOL
    assert np.all(a_got[~fluid] == 0)
    c.close()


def test_sph_full_cfg4_sampled_parity(pm, orc):
    """BJ configs[3] at full size (2,462,060 particles, dp = 1/160): sampled
    densities, and accelerations of a stratified sample (free surface, wall,
    interior) against the oracle, which gets its own densities of the sampled
    rows' whole neighbourhoods (brute force, fp64)."""
    s = inputs.cfg4(vel_key=(104,))
    assert s.n == 2462060
    p = s.params
    c = _sph_ctx(pm, s)
    st = c.get_state()
    inv_sorted = np.argsort(st["gid"])
    rng = np.random.default_rng(5)
    rows = rng.choice(s.n, 200, replace=False)
    rho_ref, _ = orc.sph_density_rows(s.pos, s.lo, s.hi, s.periodic, p, rows=rows)
    got = st["rho"][inv_sorted[s.gid[rows]]]
    assert np.max(np.abs(got - rho_ref)) / np.sqrt(np.mean(rho_ref ** 2)) <= TOL
    x = s.pos[:, :3]
    dp = p["dp"]
    fluid = s.kind == 0
    surf = np.where(fluid & (x[:, 2] > 0.5 - 2 * dp))[0]
    wall = np.where(fluid & (x[:, 0] < 2 * dp))[0]
    inner = np.where(fluid & np.all(np.abs(x - [0.5, 0.5, 0.25]) < 0.1, axis=1))[0]
    sample = np.concatenate([rng.choice(g, 12, replace=False) for g in (surf, wall, inner)])
    rp, cols, _ = orc.verlet_rows(s.pos, s.lo, s.hi, s.periodic,
                                  np.float32(2 * np.float32(p["h"])), rows=sample,
                                  want_shift=False)
    need = np.unique(np.concatenate([sample, cols]))
    rho_n, P_n = orc.sph_density_rows(s.pos, s.lo, s.hi, s.periodic, p, rows=need)
    rho_all = np.full(s.n, np.nan)
    P_all = np.full(s.n, np.nan)
    rho_all[need] = rho_n
    P_all[need] = P_n
    a_ref = orc.sph_accel_rows(s.pos, s.vel, rho_all, P_all, s.kind, s.lo, s.hi, s.periodic, p,
                               rows=sample)
    assert np.all(np.isfinite(a_ref))
    g = np.asarray(p["g"])
    a_got = st["force"][inv_sorted[s.gid[sample]], :3].astype(np.float64)
    assert orc.normalized_max_err(a_got - g, a_ref - g) <= TOL
    c.close()


def test_sph_hydrostatic_exact_lattice(pm):
    """On a lattice exactly representable in fp32 (dp = 1/64), interior fluid
    particles at rest feel exactly g up to fp32 rounding: sum_q grad W = 0
    (pinned for the oracle in test_oracle_pins.py)."""
    s = inputs.cfg4(dp=1.0 / 64.0)
    p = s.params
    c = _sph_ctx(pm, s)
    st = c.get_state()
    x = st["pos"][:, :3]
    dp = p["dp"]
    interior = (st["gid"] >= 0) & (s.kind[st["gid"]] == 0) & np.all(x > 4 * dp, axis=1) & \
        (x[:, 0] < 1 - 6 * dp) & (x[:, 1] < 1 - 4 * dp) & (x[:, 2] < 0.5 - 6 * dp)
    a = st["force"][interior, :3].astype(np.float64)
    assert interior.sum() > 10000
    assert np.max(np.abs(a - np.asarray(p["g"]))) < 1e-3
    c.close()


# ---------------------------------------------------------------- errors / edges
def test_error_paths(pm):
    s = inputs.cfg1()
    # coincident pair
    s2 = s.subset(np.arange(s.n))
    s2.pos[1, :3] = s2.pos[0, :3]
    c = make_ctx(pm, s2)
    with pytest.raises(pm.PMError) as e:
        c.build_verlet()
    assert e.value.code == -7
    c.close()
    # coincident pair in a sparse grid (lane-per-cell sort) and in a crowded
    # cell of it (the warp path inside the same kernel)
    for k0, k1, crowd in ((0, 1, 0), (2, 3, 20)):
        s4 = inputs.random_box(3000, 40.0, (18,))
        if crowd:
            s4.pos[:crowd, :3] = np.random.default_rng(9).uniform(20.0, 22.7, (crowd, 3))
        s4.pos[k1, :3] = s4.pos[k0, :3]
        c = make_ctx(pm, s4)
        with pytest.raises(pm.PMError) as e:
            c.build_verlet()
        assert e.value.code == -7
        c.close()
    # coincident pair inside a cell of more than 32 members (block-level sort,
    # no pairwise check there): the force sweep raises PM_E_COINCIDENT
    s5 = inputs.random_box(3000, 40.0, (19,))
    s5.pos[:60, :3] = np.random.default_rng(10).uniform(20.0, 22.5, (60, 3))
    s5.pos[7, :3] = s5.pos[3, :3]
    c = make_ctx(pm, s5)
    c.build_verlet()
    with pytest.raises(pm.PMError) as e:
        c.compute_lj()
    assert e.value.code == -7
    c.close()
    # outside a non-periodic axis
    s3 = s.subset(np.arange(s.n))
    s3.periodic = np.array([1, 1, 0], np.int32)
    s3.pos[5, 2] = -1.0
    c = make_ctx(pm, s3)
    with pytest.raises(pm.PMError) as e:
        c.build_cells()
    assert e.value.code == -6
    c.close()
    # periodic box shorter than 3 r_v
    c = pm.Context()
    with pytest.raises(pm.PMError) as e:
        c.set_domain([0, 0, 0], [8, 8, 8], [1, 1, 1])
        c.set_cutoff(2.5, 0.3)
    assert e.value.code == -1
    c.close()
    # forces before a list
    c = make_ctx(pm, s)
    with pytest.raises(pm.PMError) as e:
        c.compute_lj()
    assert e.value.code == -2
    c.close()


def test_tiny_and_ragged_sizes(pm, orc):
    """n not a multiple of 32 / 256, and a single particle (empty rows)."""
    for n in (1, 33, 1000, 4097):
        s = inputs.random_box(n, 9.0, (20, n))
        c = make_ctx(pm, s, r_min=0.8)  # capped: random clouds have close pairs
        c.build_verlet()
        c.compute_lj()
        st = c.get_state()
        inv = idx_of_gid(s)
        ref = orc.lj_rows(s.pos, s.lo, s.hi, s.periodic, rc=2.5, r_min=0.8,
                          rows=inv[st["gid"]])
        if n > 1:
            assert orc.normalized_max_err(st["force"][:, :3], ref["F"]) <= TOL
        else:
            assert np.all(st["force"] == 0)
        c.close()


def test_empty_inputs(pm):
    """Zero particles: before any placement the calls report PM_E_STATE; a
    context emptied by pm_place(n = 0) builds, sweeps and steps nothing
    (every launcher guards n = 0) and returns empty arrays."""
    s = inputs.cfg1()
    empty = np.zeros((0, 4), np.float32)
    c = pm.Context()
    c.set_domain(s.lo, s.hi, s.periodic)
    c.set_cutoff(2.5, 0.3)
    c.set_lj(1.0, 1.0, 1.0, 0.0)
    with pytest.raises(pm.PMError) as e:
        c.build_verlet()
    assert e.value.code == -2
    # an empty placement is a valid (empty) system: an empty sub-domain of a
    # decomposition must build and step
    c.place(empty, empty, np.zeros(0, np.int64))
    c.build_verlet()
    assert c.step_vv(0.005, 2)["steps"] == 2
    c.place(s.pos, s.vel, s.gid)
    c.build_verlet()
    c.place(empty, empty, np.zeros(0, np.int64))
    c.build_verlet()
    c.compute_lj(want_energy=True)
    r = c.step_vv(0.005, 3)
    assert r["steps"] == 3 and r["rebuilds"] == 0
    assert c.count()["nnz"] == 0
    st = c.get_state()
    assert st["pos"].shape == (0, 4) and st["gid"].shape == (0,)
    rp, col = c.get_verlet()
    assert rp.tolist() == [0] and col.size == 0
    assert c.thermo()["npairs"] == 0
    c.close()
    # SPH stepping and DEM on an emptied context
    s4 = inputs.cfg4(dp=1.0 / 16.0)
    c = pm.Context()
    c.set_domain(s4.lo, s4.hi, s4.periodic)
    c.set_cutoff(2.0 * s4.params["h"], 0.1 * s4.params["h"])
    c.set_sph(s4.params)
    c.place(s4.pos, s4.vel, s4.gid, s4.kind)
    c.place(empty, empty, np.zeros(0, np.int64), np.zeros(0, np.int32))
    assert c.sph_run(5)["steps"] == 5
    c.close()
    s5 = inputs.dem_avalanche(4, 4, 4)
    c = pm.Context()
    c.set_domain(s5.lo, s5.hi, s5.periodic)
    c.set_cutoff(2.0 * s5.params["R"], s5.params["skin"])
    c.set_dem(s5.params)
    c.place(s5.pos, s5.vel, s5.gid)
    c.place(empty, empty, np.zeros(0, np.int64))
    assert c.dem_run(s5.params["dt"], 5) == 0
    c.close()


def hydrostatic_rho(z, p):
    """Initial density of a fluid column at rest (the DualSPHysics dam-break
    start): P = rho0 |g| (h_swl - z) for z < h_swl, rho = rho0 (1 + P/b)^(1/gamma)
    (the Tait EOS Eq. 3 inverted); rho0 above the surface."""
    P = p["rho0"] * 9.81 * np.maximum(p["h_swl"] - np.asarray(z, np.float64), 0.0)
    return (p["rho0"] * (1.0 + P / p["b"]) ** (1.0 / p["gamma"])).astype(np.float32)


def test_sph_run_parity_small_dam(pm, orc):
    """WCSPH time stepping (pm_sph_run, readings R26-R28)
    against the fp64 oracle (oracle.sph_run): a dp = 1/16 dam-break block
    with a hydrostatic initial density, 30 Verlet steps with dynamic dt and an
    Euler step every 10.  fp32 state on the GPU, fp64 in the oracle: dt per
    step, positions, velocities and densities must agree closely over this
    short horizon."""
    s = inputs.cfg4(dp=1.0 / 16.0)
    p = s.params
    c = pm.Context()
    c.set_domain(s.lo, s.hi, s.periodic)
    c.set_cutoff(2.0 * p["h"], 0.1 * p["h"])
    c.set_sph(p)
    c.place(s.pos, s.vel, s.gid, s.kind)
    c.build_verlet()
    st0 = c.get_state()
    c.set_rho(hydrostatic_rho(st0["pos"][:, 2], p))
    rho_init = hydrostatic_rho(s.pos[:, 2], p).astype(np.float64)
    nsteps = 30
    r = c.sph_run(nsteps, cfl=0.2, every=10)
    assert r["steps"] == nsteps
    st = c.get_state()
    order = np.argsort(st["gid"])
    x_ref, v_ref, rho_ref, dt_ref = orc.sph_run(s.pos, s.vel, rho_init, s.kind, s.lo, s.hi,
                                                s.periodic, p, nsteps, cfl=0.2, every=10)
    assert r["time"] == pytest.approx(dt_ref.sum(), rel=1e-4)
    assert r["dt_min"] == pytest.approx(dt_ref.min(), rel=1e-4)
    x = st["pos"][order, :3].astype(np.float64)
    v = st["vel"][order, :3].astype(np.float64)
    rho = st["rho"][order].astype(np.float64)
    assert np.max(np.abs(x - x_ref)) < 1e-4 * p["dp"]
    vscale = max(np.max(np.abs(v_ref)), 1e-12)
    assert np.max(np.abs(v - v_ref)) / vscale < 1e-3
    assert np.max(np.abs(rho - rho_ref) / p["rho0"]) < 1e-5
    # boundary particles did not move
    b = s.kind == 1
    assert np.array_equal(st["pos"][order][b, :3], s.pos[b, :3])
    c.close()


def test_dem_parity_granular_packing(pm, orc):
    """DEM (pm_dem_run, Eqs. 9-13, readings
    R29-R33) against the fp64 oracle: 800 grains with walls, periodic y,
    gravity, friction; after 200 and 1000 steps (the latter with ~20 Verlet
    rebuilds that carry the contact histories over by gid) positions,
    velocities and spins follow the oracle up to fp32 drift; a smaller skin
    (more rebuilds) gives the same trajectory."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location(
        "dem_check", os.path.join(os.path.dirname(__file__), "..", "tools", "dem_check.py"))
    dc = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(dc)
    P = dc.P
    pos, vel, gid, lo, hi, per = dc.granular()

    def gpu(nsteps, skin):
        c = pm.Context()
        c.set_domain(lo, hi, per)
        c.set_cutoff(2 * P["R"], skin)
        c.set_dem(P)
        c.place(pos, vel, gid)
        reb = c.dem_run(2e-4, nsteps)
        st = c.get_state()
        w = c.get_dem()["omega"]
        o = np.argsort(st["gid"])
        c.close()
        return st["pos"][o, :3].astype(np.float64), st["vel"][o, :3].astype(np.float64), \
            w[o, :3].astype(np.float64), reb

    for nsteps, tx, tv, tw in ((200, 1e-3, 2e-3, 2e-2), (1000, 5e-3, 5e-3, 2e-2)):
        x, v, w, reb = gpu(nsteps, 0.02)
        xr, vr, wr, _ = orc.dem_run(pos, vel, np.zeros_like(pos), gid, lo, hi, per, P["walls"], P,
                                    2e-4, nsteps)
        assert np.max(np.abs(x - xr)) / P["R"] < tx
        assert np.max(np.abs(v - vr)) / np.max(np.abs(vr)) < tv
        assert np.max(np.abs(w - wr)) / np.max(np.abs(wr)) < tw
        if nsteps == 1000:
            assert reb >= 10
            x2, v2, w2, reb2 = gpu(nsteps, 0.008)
            assert reb2 > reb
            assert np.max(np.abs(x2 - x)) / P["R"] < tx
            assert np.max(np.abs(w2 - w)) / np.max(np.abs(wr)) < tw


def _dem_ctx(pm, s):
    p = s.params
    c = pm.Context()
    c.set_domain(s.lo, s.hi, s.periodic)
    c.set_cutoff(2.0 * p["R"], p["skin"])
    c.set_dem(p)
    c.place(s.pos, s.vel, s.gid)
    return c


def test_dem_avalanche_small_parity(pm, orc):
    """The avalanche recipe (inputs.dem_avalanche, reading R34)
    at 12 x 8 x 6 grains: tilted gravity, x walls and floor, periodic y;
    300 steps from the lattice (the column compresses and starts to slide)
    against the fp64 oracle."""
    s = inputs.dem_avalanche(12, 8, 6)
    p = s.params
    c = _dem_ctx(pm, s)
    c.dem_run(p["dt"], 300)
    st = c.get_state()
    w = c.get_dem()["omega"]
    o = np.argsort(st["gid"])
    c.close()
    xr, vr, wr, nh = orc.dem_run(s.pos, s.vel, np.zeros_like(s.pos), s.gid, s.lo, s.hi,
                                 s.periodic, p["walls"], p, p["dt"], 300)
    assert nh > s.n  # a dense contact network formed
    assert np.max(np.abs(st["pos"][o, :3] - xr)) / p["R"] < 1e-3
    assert np.max(np.abs(st["vel"][o, :3] - vr)) / np.max(np.abs(vr)) < 2e-3
    assert np.max(np.abs(w[o, :3] - wr)) / np.max(np.abs(wr)) < 2e-2


def test_dem_avalanche_full_size_momentum(pm):
    """Full size (679,140 grains, the bench's DEM workload): the ordered-pair
    forces are exact negatives of each other (exactly negated r_pq, n, v_pq
    and histories) and walls push only along x and z, so the y momentum
    changes by accumulation rounding only; every grain stays inside."""
    s = inputs.dem_avalanche()
    p = s.params
    c = _dem_ctx(pm, s)
    py0 = s.vel[:, 1].astype(np.float64).sum()
    reb = c.dem_run(p["dt"], 400)
    st = c.get_state()
    c.close()
    assert st["gid"].shape[0] == s.n and np.array_equal(np.sort(st["gid"]), s.gid)
    py1 = st["vel"][:, 1].astype(np.float64).sum()
    impulse = s.n * 9.81 * p["dt"] * 400  # |g| t N m: the scale of the x/z momentum change
    assert abs(py1 - py0) < 1e-6 * impulse, (py0, py1)
    assert np.all(st["pos"][:, :3] >= s.lo) and np.all(st["pos"][:, :3] < s.hi)
    assert reb >= 0


def test_dem_graph_matches_host_loop_with_resume(pm):
    """pm_dem_run's CUDA graph (conditional rebuild node, no host round trip
    per step) gives bit-identical trajectories to the plain host loop (same
    kernels, same order), including a resume after a neighbour-capacity
    overflow inside the graph: the initial rows of the lattice avalanche fit
    8 slots (bulk rows 6), the collapsing packing needs more."""
    s = inputs.dem_avalanche(12, 8, 10)
    p = s.params

    def run(graphs):
        c = pm.Context(nbr_cap=8, use_graphs=graphs)
        c.set_domain(s.lo, s.hi, s.periodic)
        c.set_cutoff(2.0 * p["R"], p["skin"])
        c.set_dem(p)
        c.place(s.pos, s.vel, s.gid)
        c.build_verlet()
        rp0, _ = c.get_verlet()
        reb = c.dem_run(p["dt"], 1500)
        st = c.get_state()
        w = c.get_dem()["omega"]
        rp1, _ = c.get_verlet()
        c.close()
        return st, w, reb, np.diff(rp0).max(), np.diff(rp1).max()

    a = run(True)
    b = run(False)
    assert a[3] <= 8 and a[4] > 8  # the list outgrew the first layout inside the graph
    assert a[2] == b[2] and a[2] > 0
    for k in ("pos", "vel", "gid"):
        assert np.array_equal(a[0][k], b[0][k]), k
    assert np.array_equal(a[1], b[1])


def test_largest_config_size_uniform(pm, orc):
    """The largest particle count of the BASELINE configs (cfg5's 8,388,608)
    on one context, as a uniform rho = 0.8 liquid (256 x 256 x 128 SC
    lattice; cfg5's clustered layout needs the 8-GPU split): cells bit-exact
    on sampled particles, sampled Verlet rows and forces against the oracle,
    and 5 steps through the step graph."""
    s = inputs.lj_lattice_system(256, 256, 128, jitter_key=(77,), vel_key=(177,))
    assert s.n == 8388608
    c = make_ctx(pm, s)
    c.build_verlet()
    rp, col = c.get_verlet()
    st = c.get_state()
    inv = idx_of_gid(s)
    pick = np.random.default_rng(4).choice(s.n, 120, replace=False)
    rrp, rcols, _ = orc.verlet_rows(s.pos, s.lo, s.hi, s.periodic, rv32(2.5, 0.3),
                                    rows=inv[st["gid"][pick]], want_shift=False)
    for t, i in enumerate(pick):
        assert np.array_equal(np.sort(col[rp[i]:rp[i + 1]]),
                              np.sort(s.gid[rcols[rrp[t]:rrp[t + 1]]])), f"row {i}"
    c.compute_lj()
    st = c.get_state()
    ref = orc.lj_rows(s.pos, s.lo, s.hi, s.periodic, rc=2.5, rows=inv[st["gid"][pick]])
    assert orc.normalized_max_err(st["force"][pick, :3].astype(np.float64), ref["F"]) <= TOL
    r = c.step_vv(0.005, 5)
    assert r["steps"] == 5
    c.close()


def test_sph_run_graph_equals_host_loop(pm):
    """pm_sph_run's CUDA graph (conditional rebuild node; dt, Euler steps and
    the rebuild decision all on the device) gives bit-identical states to the
    plain host loop, rebuilds included."""
    s = inputs.cfg4(dp=1.0 / 16.0, vel_key=(105,), vmax=0.5)
    p = s.params
    out = []
    for graphs in (True, False):
        c = pm.Context(use_graphs=graphs)
        c.set_domain(s.lo, s.hi, s.periodic)
        c.set_cutoff(2.0 * p["h"], 0.1 * p["h"])
        c.set_sph(p)
        c.place(s.pos, s.vel, s.gid, s.kind)
        c.build_verlet()
        c.set_rho(hydrostatic_rho(c.get_state()["pos"][:, 2], p))
        r = c.sph_run(120, cfl=0.2, every=10)
        out.append((c.get_state(), r))
        c.close()
    (a, ra), (b, rb) = out
    assert ra["steps"] == rb["steps"] == 120 and ra["rebuilds"] == rb["rebuilds"] >= 1
    assert ra["time"] == rb["time"]
    for k in ("pos", "vel", "rho", "gid"):
        assert np.array_equal(a[k], b[k]), k


def test_set_lj_flags_contract(pm):
    """pm_set_lj(flags, r_min): PM_LJ_CAPPED needs r_min > 0,
    the plain potential r_min = 0, unknown flags are PM_E_INVAL."""
    c = pm.Context()
    L = pm.lib()
    assert L.pm_set_lj(c.h, 1.0, 1.0, 1.0, 0, 0.0) == 0
    assert L.pm_set_lj(c.h, 1.0, 1.0, 1.0, pm.PM_LJ_CAPPED, 0.8) == 0
    assert L.pm_set_lj(c.h, 1.0, 1.0, 1.0, pm.PM_LJ_CAPPED, 0.0) == -1
    assert L.pm_set_lj(c.h, 1.0, 1.0, 1.0, 0, 0.8) == -1
    assert L.pm_set_lj(c.h, 1.0, 1.0, 1.0, 4, 0.0) == -1
    assert L.pm_set_lj(c.h, -1.0, 1.0, 1.0, 0, 0.0) == -1
    c.close()


@pytest.mark.parametrize("seed", list(range(12)))
def test_verlet_randomised_boxes_and_clusters(pm, orc, seed):
    """Randomised stress of the staged build (bounding-box culling, seam
    pieces with own / candidate shifts, per-pair R4 rows, shared-memory and
    direct rows): random box shapes from 3 r_v to 8 r_v per axis, random
    periodicity, uniform or clustered (a dense blob over a dilute gas, up to
    ~200 per cell) particles, some placed on faces and at hi - ulp; every row
    equals the oracle's O(N^2) set, and the list is symmetric."""
    rng = np.random.default_rng(1000 + seed)
    rv = float(rv32(2.5, 0.3))
    ext = rng.uniform(3.05, 8.0, 3) * rv
    per = rng.integers(0, 2, 3).astype(np.int32)
    n = int(rng.integers(300, 2500))
    x = rng.uniform(0.0, 1.0, (n, 3)) * ext
    if seed % 3 == 0:  # a dense cluster
        m = n // 3
        x[:m] = ext * 0.5 + rng.normal(0.0, 0.6, (m, 3))
        x = np.clip(x, 0.0, ext * (1 - 1e-6))
    if seed % 4 == 1:  # faces and hi - ulp
        k = n // 10
        ax = rng.integers(0, 3, k)
        x[np.arange(k), ax] = np.where(rng.random(k) < 0.5, 0.0,
                                       np.nextafter(np.float32(ext[ax]), np.float32(0)))
    pos = np.zeros((n, 4), np.float32)
    pos[:, :3] = x.astype(np.float32)
    hi = ext.astype(np.float32)
    pos[:, :3] = np.minimum(pos[:, :3], np.nextafter(hi, np.float32(0)))
    s = inputs.System(pos=pos, vel=np.zeros_like(pos), gid=np.arange(n, dtype=np.int64),
                      lo=np.zeros(3, np.float32), hi=hi, periodic=per, params={})
    c = make_ctx(pm, s)
    c.build_verlet()
    rp, col = c.get_verlet()
    st = c.get_state()
    rrp, rcols, _ = orc.verlet_rows(s.pos, s.lo, s.hi, s.periodic, rv32(2.5, 0.3),
                                    rows=st["gid"], want_shift=False)
    bad = _row_sets_equal(rp, col, st["gid"], rrp, rcols, s.gid)
    assert bad < 0, f"row {bad} differs (seed {seed})"
    # symmetry of the gid pair sets
    rows = np.repeat(st["gid"], np.diff(rp))
    a = set(zip(rows.tolist(), col.tolist()))
    assert all((j, i) in a for (i, j) in a)
    c.close()
