"""Multi-GPU path on ONE GPU (in-process loopback transport): the same global
system run whole on one context and decomposed into P sub-domains must give
identical neighbour sets (as gid pairs), the same forces (1e-4 of RMS; the
pair sets are identical so only summation order differs) and, over a short
run with rebuilds and migrations, the same trajectory (SURVEY §8(c)
"Multi-GPU: rank-count independence", §4 T3)."""
import numpy as np
import pytest

from paper_1804_07598_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1804_07598_b200 import build, dist, pm
    build.build()
    return pm, dist


def single(pm, s):
    c = pm.Context()
    c.set_domain(s.lo, s.hi, s.periodic)
    c.set_cutoff(2.5, 0.3)
    c.set_lj(1.0, 1.0, 1.0, 0.0)
    c.place(s.pos, s.vel, s.gid)
    return c


def decomposed(pm, dist, s, grid):
    import torch
    D = dist.Decomp(grid)
    owner = dist.owner_of(s, D)
    stream = torch.cuda.Stream()
    members = {}
    for r in range(D.size):
        sub = s.subset(np.where(owner == r)[0])
        members[r] = dist.make_member(sub, D, r, stream=stream)
    sim = dist.DistSim(D, members, dist.LoopbackTransport(members), stream=stream)
    return sim


def owned_union(pm, sim):
    parts = [ctx.owned_state() for ctx in sim.m.values()]
    st = {k: np.concatenate([p[k] for p in parts]) for k in parts[0]}
    return pm.sorted_by_gid(st)


@pytest.mark.parametrize("grid", [(2, 1, 1), (2, 2, 1), (2, 2, 2), (3, 1, 2)])
def test_decomposed_lists_and_forces_match_single(env, grid):
    pm, dist = env
    s = inputs.lj_lattice_system(18, 18, 18, jitter_key=(41,), vel_key=(141,))
    ref = single(pm, s)
    ref.build_verlet()
    ref.compute_lj()
    rst = pm.sorted_by_gid(ref.get_state())
    rrp, rcol = ref.get_verlet()
    rgid = ref.get_state()["gid"]
    ref_rows = {int(g): set(rcol[rrp[i]:rrp[i + 1]].tolist()) for i, g in enumerate(rgid)}
    sim = decomposed(pm, dist, s, grid)
    sim.start()
    got = owned_union(pm, sim)
    assert np.array_equal(got["gid"], np.sort(s.gid))  # every particle owned exactly once
    F, Fr = got["force"][:, :3].astype(np.float64), rst["force"][:, :3].astype(np.float64)
    err = np.max(np.abs(F - Fr)) / np.sqrt(np.mean(Fr ** 2))
    assert err <= 1e-4, err
    # neighbour sets as gid sets, row by row (owned rows only)
    for ctx in sim.m.values():
        rp, col = ctx.get_verlet()
        st = ctx.get_state()
        kind = ctx.kind()
        for i in range(len(st["gid"])):
            if kind[i] & pm.GHOST_BIT:
                assert rp[i + 1] == rp[i]
                continue
            assert set(col[rp[i]:rp[i + 1]].tolist()) == ref_rows[int(st["gid"][i])]
    ref.close()
    for ctx in sim.m.values():
        ctx.close()


@pytest.mark.parametrize("grid", [(2, 1, 1), (2, 2, 2)])
def test_decomposed_trajectory_matches_single(env, grid):
    """40 NVE steps with rebuilds, migration and ghost refresh: positions and
    velocities agree with the single-context run (fp32, summation order only)."""
    pm, dist = env
    s = inputs.lj_lattice_system(18, 18, 18, jitter_key=(42,), vel_key=(142,))
    ref = single(pm, s)
    r = ref.step_vv(0.005, 40)
    rst = pm.sorted_by_gid(ref.get_state())
    sim = decomposed(pm, dist, s, grid)
    sim.start()
    reb = sim.run(40)
    assert reb >= 2 and r["rebuilds"] >= 2
    got = owned_union(pm, sim)
    assert np.array_equal(got["gid"], np.sort(s.gid))
    L = s.hi.astype(np.float64)
    d = got["pos"][:, :3].astype(np.float64) - rst["pos"][:, :3]
    d -= L * np.round(d / L)
    assert np.max(np.abs(d)) < 1e-3
    assert np.max(np.abs(got["vel"][:, :3] - rst["vel"][:, :3])) < 1e-2
    th = sim.thermo()
    th_ref = ref.thermo()
    assert th["npairs"] == th_ref["npairs"]
    assert th["ke"] == pytest.approx(th_ref["ke"], rel=1e-4)
    assert th["pe_shift"] == pytest.approx(th_ref["pe_shift"], rel=1e-4)
    ref.close()
    for ctx in sim.m.values():
        ctx.close()


def test_decomposition_usage_errors(env):
    pm, dist = env
    s = inputs.lj_lattice_system(8, 8, 8, jitter_key=(43,))  # L = 8.6 < 2 * 2 r_v
    c = pm.DistContext()
    c.set_domain(s.lo, s.hi, s.periodic)
    c.set_cutoff(2.5, 0.3)
    with pytest.raises(pm.PMError) as e:
        c.set_decomposition((2, 1, 1), (0, 0, 0))
    assert e.value.code == -1
    c.close()


def test_bench_torchrun_two_ranks_share_one_gpu(env, tmp_path):
    """The N>1 bench path end to end under torchrun (2 ranks, gloo with host
    staging so both ranks can share the single GPU; no kernel ever waits on
    another rank): one JSON line with the whole-job value."""
    import json
    import os
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    # two ranks on one GPU: NCCL refuses a duplicate device, so this runs the
    # DistSim orchestration over gloo (the native NCCL group is covered by
    # test_gpu_group.py and test_bench_native_single_rank)
    env_ = dict(os.environ, PM_DIST_BACKEND="gloo", PM_CFG3_BLOCK="32", PM_DIST_NATIVE="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "12", "--warmup", "3"]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env_, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    b = json.loads(lines[0])
    assert b["n_gpus"] == 2 and b["config"]["n_particles"] == 2 * 32 ** 3
    assert b["value"] > 0 and b["e2e"]["value"] > 0


def test_load_balanced_cuts_clustered(env):
    """SURVEY NEXT-2 (§3.5): on a clustered system (cfg5-like,
    8 Gaussian clusters) the tensor-product cuts at weighted quantiles of the
    pair counts lower the per-sub-domain work imbalance (max/mean list
    entries) of a 2x2x2 decomposition, and the balanced decomposition gives
    the same neighbour sets and forces as one context."""
    import torch
    pm, dist = env
    s = inputs.cfg5(n_clusters=8, per_cluster=8192, sigma_c=6.0, rho=0.3, key=55)
    ref = pm.Context()
    ref.set_domain(s.lo, s.hi, s.periodic)
    ref.set_cutoff(2.5, 0.3)
    ref.set_lj(1.0, 1.0, 1.0, 0.8)
    ref.place(s.pos, s.vel, s.gid)
    ref.build_verlet()
    ref.compute_lj()
    rst = pm.sorted_by_gid(ref.get_state())
    rp, _ = ref.get_verlet()
    w = np.zeros(s.n)
    w[ref.get_state()["gid"]] = np.diff(rp)  # pair work per particle (by gid)
    rv = np.float32(2.8)

    def run(D):
        owner = dist.owner_of(s, D)
        stream = torch.cuda.Stream()
        members = {r: dist.make_member(s.subset(np.where(owner == r)[0]), D, r, stream=stream,
                                       r_min=0.8) for r in range(D.size)}
        sim = dist.DistSim(D, members, dist.LoopbackTransport(members), stream=stream)
        sim.start()
        work = [ctx.count()["nnz"] for ctx in sim.m.values()]
        got = pm.sorted_by_gid(
            {k: np.concatenate([ctx.owned_state()[k] for ctx in sim.m.values()])
             for k in ("gid", "force")})
        for ctx in sim.m.values():
            ctx.close()
        return work, got

    w_uni, _ = run(dist.Decomp((2, 2, 2)))
    Db = dist.balanced_decomp((2, 2, 2), s.pos[:, :3], w, s.lo, s.hi, float(rv))
    w_bal, got = run(Db)
    assert sum(w_uni) == sum(w_bal)  # same pairs, other owners
    assert dist.imbalance(w_bal) < dist.imbalance(w_uni)
    assert np.array_equal(got["gid"], np.sort(s.gid))
    F, Fr = got["force"][:, :3].astype(np.float64), rst["force"][:, :3].astype(np.float64)
    assert np.max(np.abs(F - Fr)) / np.sqrt(np.mean(Fr ** 2)) <= 1e-4
    ref.close()


def test_over_decomposition_hybrid_clustered(env):
    """SURVEY NEXT-2 via over-decomposition (the paper's sub-sub-domains,
    PAPER.md:66-88, 122): a 4x4x4 grid of sub-domains on the clustered
    system, assigned to 8 ranks by LPT on the measured pair work, all run in
    this process through HybridTransport's local path: the rank loads are
    balanced and neighbour sets/forces equal the one-context run."""
    import torch
    pm, dist = env
    s = inputs.cfg5(n_clusters=8, per_cluster=8192, sigma_c=6.0, rho=0.3, key=56)
    ref = pm.Context()
    ref.set_domain(s.lo, s.hi, s.periodic)
    ref.set_cutoff(2.5, 0.3)
    ref.set_lj(1.0, 1.0, 1.0, 0.8)
    ref.place(s.pos, s.vel, s.gid)
    ref.build_verlet()
    ref.compute_lj()
    rst = pm.sorted_by_gid(ref.get_state())
    rp, _ = ref.get_verlet(cols=False)
    w = np.zeros(s.n)
    w[ref.get_state()["gid"]] = np.diff(rp)
    D = dist.Decomp((4, 4, 4))
    owner = dist.owner_of(s, D)
    work = np.bincount(owner, weights=w, minlength=D.size)
    assign = dist.lpt_assign(work, 8)
    load = np.bincount(assign, weights=work, minlength=8)
    assert dist.imbalance(load) < 1.05 < dist.imbalance(
        np.bincount(dist.owner_of(s, dist.Decomp((2, 2, 2))), weights=w, minlength=8))
    stream = torch.cuda.Stream()
    members = {r: dist.make_member(s.subset(np.where(owner == r)[0]), D, r, stream=stream,
                                   r_min=0.8) for r in range(D.size)}
    tr = dist.HybridTransport(np.zeros(D.size, np.int64), 0)  # every sub-domain local
    sim = dist.DistSim(D, members, tr, stream=stream)
    sim.start()
    got = pm.sorted_by_gid({k: np.concatenate([c.owned_state()[k] for c in sim.m.values()])
                            for k in ("gid", "force")})
    assert np.array_equal(got["gid"], np.sort(s.gid))
    F, Fr = got["force"][:, :3].astype(np.float64), rst["force"][:, :3].astype(np.float64)
    assert np.max(np.abs(F - Fr)) / np.sqrt(np.mean(Fr ** 2)) <= 1e-4
    assert sum(c.count()["nnz"] for c in sim.m.values()) == int(rp[-1])
    reb = sim.run(10)
    assert reb >= 0
    for c in sim.m.values():
        c.close()
    ref.close()


def _hydro_rho(z, p):
    P = p["rho0"] * 9.81 * np.maximum(p["h_swl"] - np.asarray(z, np.float64), 0.0)
    return (p["rho0"] * (1.0 + P / p["b"]) ** (1.0 / p["gamma"])).astype(np.float32)


@pytest.mark.parametrize("grid", [(2, 1, 1), (2, 2, 1)])
def test_decomposed_sph_stepping_matches_single(env, grid):
    """NEXT-3 multi-GPU SPH (pm_dist_sph_*): a periodic fluid layer with
    random velocities stepped 60 times (dynamic dt from the global minimum
    step bound, Euler every 10) on P sub-domains whose ghosts carry position,
    velocity, rho and P each step, against the same run on one context and
    against the fp64 oracle.  The pair sets are identical; only fp32
    summation order differs.  (Random velocities up to 0.3 m/s: several
    rebuilds with migrations within the 60 steps.)"""
    import torch
    pm, dist = env
    from oracle import oracle as orc
    s = inputs.sph_layer(vmax=0.3)
    p = s.params
    rc, skin = 2.0 * p["h"], 0.1 * p["h"]
    rho0 = _hydro_rho(s.pos[:, 2], p)
    nsteps, cfl, every = 60, 0.2, 10
    # one context
    c = pm.Context()
    c.set_domain(s.lo, s.hi, s.periodic)
    c.set_cutoff(rc, skin)
    c.set_sph(p)
    c.place(s.pos, s.vel, s.gid, s.kind)
    c.build_verlet()
    c.set_rho(_hydro_rho(c.get_state()["pos"][:, 2], p))
    r1 = c.sph_run(nsteps, cfl=cfl, every=every)
    one = pm.sorted_by_gid(c.get_state())
    c.close()
    # decomposed, loopback transport on this GPU
    D = dist.Decomp(grid)
    owner = dist.owner_of(s, D)
    stream = torch.cuda.Stream()
    members = {}
    for r in range(D.size):
        idx = np.where(owner == r)[0]
        m = dist.make_member(s.subset(idx), D, r, stream=stream, rc=rc, skin=skin, sph=p)
        m.set_rho(rho0[idx])
        members[r] = m
    sim = dist.DistSim(D, members, dist.LoopbackTransport(members), stream=stream)
    sim.sph_start()
    reb, t = sim.sph_run(nsteps, cfl=cfl, every=every)
    torch.cuda.synchronize()
    assert reb >= 2 and r1["rebuilds"] >= 2  # migrations and new ghost layers on the way
    got = owned_union(pm, sim)
    assert np.array_equal(got["gid"], s.gid)  # every particle owned exactly once
    assert t == pytest.approx(r1["time"], rel=1e-5)
    dp = p["dp"]
    x, x1 = got["pos"][:, :3].astype(np.float64), one["pos"][:, :3].astype(np.float64)
    L = (s.hi - s.lo).astype(np.float64)
    dx = x - x1
    dx[:, :2] -= L[:2] * np.round(dx[:, :2] / L[:2])  # periodic images
    assert np.max(np.abs(dx)) < 1e-4 * dp
    v, v1 = got["vel"][:, :3].astype(np.float64), one["vel"][:, :3].astype(np.float64)
    assert np.max(np.abs(v - v1)) / np.max(np.abs(v1)) < 1e-3
    assert np.max(np.abs(got["rho"].astype(np.float64) - one["rho"])) / p["rho0"] < 1e-5
    # the oracle on the same run
    xr, vr, rr, dtr = orc.sph_run(s.pos, s.vel, rho0.astype(np.float64), s.kind, s.lo, s.hi,
                                  s.periodic, p, nsteps, cfl=cfl, every=every)
    assert t == pytest.approx(dtr.sum(), rel=1e-4)
    dx = x - xr
    dx[:, :2] -= L[:2] * np.round(dx[:, :2] / L[:2])
    assert np.max(np.abs(dx)) < 1e-4 * dp
    assert np.max(np.abs(v - vr)) / np.max(np.abs(vr)) < 1e-3
    assert np.max(np.abs(got["rho"] - rr)) / p["rho0"] < 1e-5
    for m in members.values():
        m.close()


def test_cfg3_full_size_decomposed_sampled_parity(env):
    """BJ configs[2] at full size in the launch configuration of the N = 2
    bench (one 128^3 block = 2,097,152 particles per sub-domain, grid
    (2,1,1), 4.2M particles in two contexts on this GPU): every particle owned
    once, sampled rows' neighbour sets (gid pairs, ghosts included) and
    forces against the fp64 oracle on the global system, then 10 steps with
    the per-step ghost refresh."""
    pm, dist = env
    from oracle import oracle as orc
    grid = (2, 1, 1)
    s = inputs.cfg3_global(grid)
    sim = decomposed(pm, dist, s, grid)
    sim.start()
    inv = np.empty(s.n, np.int64)
    inv[s.gid] = np.arange(s.n)
    rng = np.random.default_rng(9)
    rv = np.float32(np.float32(2.5) + np.float32(0.3))
    seen = 0
    for ctx in sim.m.values():
        st = ctx.get_state()
        kind = ctx.get_kind()
        own = np.where((kind & pm.GHOST_BIT) == 0)[0]
        seen += own.size
        pick = rng.choice(own, 150, replace=False)
        rp, col = ctx.get_verlet()
        rrp, rcols, _ = orc.verlet_rows(s.pos, s.lo, s.hi, s.periodic, rv,
                                        rows=inv[st["gid"][pick]], want_shift=False)
        for t, i in enumerate(pick):
            assert np.array_equal(np.sort(col[rp[i]:rp[i + 1]]),
                                  np.sort(s.gid[rcols[rrp[t]:rrp[t + 1]]])), f"row {i}"
        ref = orc.lj_rows(s.pos, s.lo, s.hi, s.periodic, rc=2.5, rows=inv[st["gid"][pick]])
        err = orc.normalized_max_err(st["force"][pick, :3].astype(np.float64), ref["F"])
        assert err <= 1e-4, err
    assert seen == s.n
    sim.run(10)
    got = owned_union(pm, sim)
    assert np.array_equal(got["gid"], np.sort(s.gid))
    for ctx in sim.m.values():
        ctx.close()


def test_decomposed_dem_matches_single(env):
    """Decomposed DEM (pm_dist_dem_*, NEXT-4 on the §8(e) decomposition;
    PAPER.md:479): an avalanche split along its periodic y axis (1,2,1),
    500 steps with migrations that carry the grains' contact histories and
    ghosts refreshed with x, v, omega, against the same run on one context
    and against the fp64 oracle; the final-step torques (which depend on
    every tangential history) agree too."""
    import torch
    pm, dist = env
    from oracle import oracle as orc
    s = inputs.dem_avalanche(10, 12, 6, vjit=1.5, gap=0.5)  # loose, fast: grains cross y faces
    p = s.params
    nsteps = 500
    c = pm.Context()
    c.set_domain(s.lo, s.hi, s.periodic)
    c.set_cutoff(2.0 * p["R"], p["skin"])
    c.set_dem(p)
    c.place(s.pos, s.vel, s.gid)
    c.dem_run(p["dt"], nsteps)
    one = c.get_state()
    o1 = np.argsort(one["gid"])
    dm1 = c.get_dem()
    w1, t1 = dm1["omega"][o1, :3], dm1["torque"][o1, :3]
    x1, v1 = one["pos"][o1, :3].astype(np.float64), one["vel"][o1, :3].astype(np.float64)
    c.close()
    D = dist.Decomp((1, 2, 1))
    owner0 = dist.owner_of(s, D)
    stream = torch.cuda.Stream()
    members = {r: dist.make_member(s.subset(np.where(owner0 == r)[0]), D, r, stream=stream,
                                   rc=2.0 * p["R"], skin=p["skin"], dem=p)
               for r in range(D.size)}
    sim = dist.DistSim(D, members, dist.LoopbackTransport(members), stream=stream)
    sim.dem_start()
    reb = sim.dem_run(nsteps, p["dt"])
    torch.cuda.synchronize()
    parts = []
    for m in members.values():
        st = m.get_state()
        own = (m.get_kind() & pm.GHOST_BIT) == 0
        dm = m.get_dem()
        parts.append((st["gid"][own], st["pos"][own, :3], st["vel"][own, :3],
                      dm["omega"][own, :3],
                      dm["torque"][own, :3]))
    gid = np.concatenate([q[0] for q in parts])
    o = np.argsort(gid)
    assert np.array_equal(gid[o], s.gid)  # every grain owned once
    x, v, w, t = (np.concatenate([q[k] for q in parts])[o].astype(np.float64) for k in (1, 2, 3, 4))
    moved = dist.owner_of(inputs.System(pos=np.c_[x, np.zeros(len(x))].astype(np.float32),
                                        vel=s.vel, gid=s.gid, lo=s.lo, hi=s.hi,
                                        periodic=s.periodic), D) != owner0
    assert reb >= 2 and moved.sum() >= 5  # grains changed owner, histories migrated
    R = p["R"]
    L = float(s.hi[1] - s.lo[1])
    dx = x - x1
    dx[:, 1] -= L * np.round(dx[:, 1] / L)
    assert np.max(np.abs(dx)) / R < 1e-3
    assert np.max(np.abs(v - v1)) / np.max(np.abs(v1)) < 2e-3
    assert np.max(np.abs(w - w1)) / np.max(np.abs(w1)) < 2e-2
    tscale = np.sqrt(np.mean(t1.astype(np.float64) ** 2))
    assert np.max(np.abs(t - t1)) / tscale < 5e-2
    xr, vr, wr, _ = orc.dem_run(s.pos, s.vel, np.zeros_like(s.pos), s.gid, s.lo, s.hi, s.periodic,
                                p["walls"], p, p["dt"], nsteps)
    # fp32 vs fp64: the gap grows with the violence of the collisions (1.5 m/s
    # impacts here); the decomposed-vs-single comparison above is the tight one
    dx = x - xr
    dx[:, 1] -= L * np.round(dx[:, 1] / L)
    assert np.max(np.abs(dx)) / R < 1e-2
    assert np.max(np.abs(v - vr)) / np.max(np.abs(vr)) < 1e-2
    dx1 = x1 - xr
    dx1[:, 1] -= L * np.round(dx1[:, 1] / L)
    assert np.max(np.abs(dx)) < 3 * np.max(np.abs(dx1)) + 1e-6  # no worse than one context
    for m in members.values():
        m.close()


def test_api_state_errors(env):
    """Call-order and mode errors of the newer entry points report
    PM_E_STATE (-2) / PM_E_INVAL (-1) instead of running: SPH / DEM stepping
    of a decomposed context before its init, full-list step phases on half
    lists, SPH and DEM on half lists, the record size of an unknown kind."""
    pm, dist = env
    s = inputs.lj_lattice_system(16, 16, 16, jitter_key=(44,))
    D = dist.Decomp((2, 1, 1))
    m = dist.make_member(s.subset(np.where(dist.owner_of(s, D) == 0)[0]), D, 0)
    for call, code in ((lambda: m.dist_sph_rates(), -2),
                       (lambda: m.dist_sph_update(1e-4), -2), (lambda: m.dist_dem_step(1e-4), -2),
                       (lambda: m.dist_dem_init(), -2)):
        with pytest.raises(pm.PMError) as e:
            call()
        assert e.value.code == code
    m.set_newton(True)  # decomposed half lists step in the NEWTON_* phases only
    with pytest.raises(pm.PMError) as e:
        m.dist_step(0.005, pm.PM_PHASE_STEP)
    assert e.value.code == -2
    m.close()
    assert pm.record_bytes(6) == -1 and pm.record_bytes(-1) == -1
    assert [pm.record_bytes(k) for k in range(6)] == [64, 32, 16, 32, 48, 592]
    c = pm.Context()
    c.set_newton(True)
    c.set_domain(s.lo, s.hi, s.periodic)
    c.set_cutoff(2.5, 0.3)
    c.set_sph(inputs.cfg4(dp=1.0 / 16.0).params)
    c.place(s.pos, s.vel, s.gid)
    with pytest.raises(pm.PMError) as e:
        c.sph_run(2)
    assert e.value.code == -2
    c.close()


def test_decomposed_dem_2x2_periodic_layer(env):
    """Decomposed DEM on a (2,2,1) grid: a granular layer periodic in x and y
    on a floor (walls only at z-lo), gravity tilted along x so grains flow
    across the x faces and collide across the y faces; histories migrate in
    all in-plane directions including the diagonals.  Matches one context."""
    import torch
    pm, dist = env
    s = inputs.dem_avalanche(12, 12, 5, vjit=1.5, gap=0.5)
    s.periodic = np.array([1, 1, 0], np.int32)
    s.hi[0] = np.float32(12 * 2 * 0.06 * 1.5)  # periodic x: the lattice length
    p = dict(s.params)
    p["walls"] = (0, 0, 0, 0, 1, 0)
    nsteps = 400
    c = pm.Context()
    c.set_domain(s.lo, s.hi, s.periodic)
    c.set_cutoff(2.0 * p["R"], p["skin"])
    c.set_dem(p)
    c.place(s.pos, s.vel, s.gid)
    c.dem_run(p["dt"], nsteps)
    one = pm.sorted_by_gid(c.get_state())
    c.close()
    D = dist.Decomp((2, 2, 1))
    owner0 = dist.owner_of(s, D)
    stream = torch.cuda.Stream()
    members = {r: dist.make_member(s.subset(np.where(owner0 == r)[0]), D, r, stream=stream,
                                   rc=2.0 * p["R"], skin=p["skin"], dem=p)
               for r in range(D.size)}
    sim = dist.DistSim(D, members, dist.LoopbackTransport(members), stream=stream)
    sim.dem_start()
    reb = sim.dem_run(nsteps, p["dt"])
    torch.cuda.synchronize()
    got = pm.sorted_by_gid({k: np.concatenate([m.owned_state()[k] for m in members.values()])
                            for k in ("gid", "pos", "vel")})
    assert np.array_equal(got["gid"], s.gid)
    own1 = dist.owner_of(inputs.System(pos=got["pos"], vel=s.vel, gid=s.gid, lo=s.lo, hi=s.hi,
                                       periodic=s.periodic), D)
    assert reb >= 2 and (own1 != owner0).sum() >= 5
    L = (s.hi - s.lo).astype(np.float64)
    dx = got["pos"][:, :3].astype(np.float64) - one["pos"][:, :3]
    dx[:, :2] -= L[:2] * np.round(dx[:, :2] / L[:2])
    assert np.max(np.abs(dx)) / p["R"] < 1e-3
    v1 = one["vel"][:, :3].astype(np.float64)
    assert np.max(np.abs(got["vel"][:, :3] - v1)) / np.max(np.abs(v1)) < 2e-3
    for m in members.values():
        m.close()


@pytest.mark.parametrize("grid", [(2, 1, 1), (2, 2, 2)])
def test_fused_ghost_refresh_matches_message_refresh(env, grid):
    """The fused ghost refresh (pm_dist_peer_setup: the sweep's epilogue
    stores every new position of a sent particle straight into the peers'
    ghost slots, no pack / message / unpack) gives bit-identical trajectories
    to the message-based refresh, over 40 steps with rebuilds and migration."""
    import torch
    pm, dist = env
    s = inputs.lj_lattice_system(18, 18, 18, jitter_key=(45,), vel_key=(145,))
    out = []
    for peer in (False, True):
        D = dist.Decomp(grid)
        owner = dist.owner_of(s, D)
        stream = torch.cuda.Stream()
        members = {r: dist.make_member(s.subset(np.where(owner == r)[0]), D, r, stream=stream)
                   for r in range(D.size)}
        sim = dist.DistSim(D, members, dist.LoopbackTransport(members), stream=stream, peer=peer)
        sim.start()
        reb = sim.run(40)
        torch.cuda.synchronize()
        out.append((owned_union(pm, sim), reb))
        for m in members.values():
            m.close()
    (a, ra), (b, rb) = out
    assert ra == rb and ra >= 2
    for k in ("gid", "pos", "vel", "force"):
        assert np.array_equal(a[k], b[k]), k


def test_bench_single_gpu_contract(env, tmp_path):
    """`python bench.py` at N = 1 (short run): one JSON line with the
    contract's keys -- whole-job value, roofline of the dominant kernel with
    its fraction of the measured peak, e2e through host buffers, launch
    count, clocks."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--steps", "30",
                        "--warmup", "3", "--no-cpu-baseline", "--no-extras"],
                       capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    b = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "config", "roofline", "e2e",
              "gpu_launches", "clocks"):
        assert k in b, k
    assert b["n_gpus"] == 1 and b["steps"] == 30 and b["value"] > 1e9
    rf = b["roofline"]
    assert rf["bound"] == "hbm" and 0.1 < rf["frac"] < 1.0 and rf["achieved"] > 0
    assert b["e2e"]["h2d_bytes_per_step"] > 0 and b["e2e"]["d2h_bytes_per_step"] > 0
    assert b["gpu_launches"] >= 2 * 30


@pytest.mark.parametrize("grid", [(2, 1, 1), (2, 2, 2)])
def test_decomposed_newton_lists_with_ghost_put(env, grid):
    """Half (Newton) lists across sub-domains (NEXT-1 with ghost_put): every
    pair -- also across a face -- is computed on exactly one rank (owned
    partners later in the local order, ghost partners with a larger gid), the
    ghosts' force shares go back to their owners.  Forces match the
    single-context full-list forces, the global pair count equals it exactly
    (each pair counted twice as ordered pairs), and 40 steps with rebuilds and
    migration follow the full-list trajectory."""
    import torch
    pm, dist = env
    s = inputs.lj_lattice_system(18, 18, 18, jitter_key=(46,), vel_key=(146,))
    ref = single(pm, s)
    ref.build_verlet()
    ref.compute_lj(want_energy=True)
    rst = pm.sorted_by_gid(ref.get_state())
    th_ref = ref.thermo(recompute=False)
    D = dist.Decomp(grid)
    owner = dist.owner_of(s, D)
    stream = torch.cuda.Stream()
    members = {r: dist.make_member(s.subset(np.where(owner == r)[0]), D, r, stream=stream)
               for r in range(D.size)}
    sim = dist.DistSim(D, members, dist.LoopbackTransport(members), stream=stream, newton=True)
    sim.start()
    torch.cuda.synchronize()
    got = owned_union(pm, sim)
    F, Fr = got["force"][:, :3].astype(np.float64), rst["force"][:, :3].astype(np.float64)
    assert np.max(np.abs(F - Fr)) / np.sqrt(np.mean(Fr ** 2)) <= 1e-4
    th = sim.thermo()
    assert th["npairs"] == th_ref["npairs"]
    assert th["pe_shift"] == pytest.approx(th_ref["pe_shift"], rel=1e-5)
    got = owned_union(pm, sim)  # forces restored after the energy pass
    assert np.max(np.abs(got["force"][:, :3] - Fr)) / np.sqrt(np.mean(Fr ** 2)) <= 1e-4
    r1 = ref.step_vv(0.005, 40)
    reb = sim.run(40)
    torch.cuda.synchronize()
    assert reb >= 2 and r1["rebuilds"] >= 2
    got = owned_union(pm, sim)
    rst = pm.sorted_by_gid(ref.get_state())
    L = s.hi.astype(np.float64)
    d = got["pos"][:, :3].astype(np.float64) - rst["pos"][:, :3]
    d -= L * np.round(d / L)
    assert np.max(np.abs(d)) < 1e-3
    assert np.max(np.abs(got["vel"][:, :3] - rst["vel"][:, :3])) < 1e-2
    ref.close()
    for m in members.values():
        m.close()


def test_runtime_rebalance_sar_clustered(env):
    """SURVEY NEXT-2 at run time (§3.5 "dynamic load
    balancing", SAR [56]): a clustered system (8 Gaussian clusters, capped LJ,
    velocity limit -- reading R22) starts on EQUAL cuts of a 2x2x2 loopback
    decomposition; DistSim.run with Stop-At-Rise re-balancing records the
    per-rank sweep times, re-cuts from all-reduced pair-work histograms (no
    gather) and migrates mid-run.  After the run: at least one re-balance,
    lower work imbalance than the equal cuts, every particle owned once, and
    sampled rows' forces equal the fp64 oracle on the global system."""
    import torch
    pm, dist = env
    from oracle import oracle as orc
    s = inputs.cfg5(n_clusters=8, per_cluster=8192, sigma_c=6.0, rho=0.3, key=57)
    D = dist.Decomp((2, 2, 2))
    owner = dist.owner_of(s, D)
    stream = torch.cuda.Stream()
    members = {r: dist.make_member(s.subset(np.where(owner == r)[0]), D, r, stream=stream,
                                   r_min=0.8) for r in range(D.size)}
    for ctx in members.values():
        ctx.set_vlimit(0.15 / 0.005)
    sim = dist.DistSim(D, members, dist.LoopbackTransport(members), stream=stream)
    sim.start()
    work0 = [ctx.count()["nnz"] for ctx in sim.m.values()]
    sim.enable_rebalance(cost_ms=0.0)
    sim.run(30)
    assert sim.rebalances >= 1
    assert sim.D.cuts is not None
    work1 = [ctx.count()["nnz"] for ctx in sim.m.values()]
    assert dist.imbalance(work1) < dist.imbalance(work0)
    got = owned_union(pm, sim)
    assert np.array_equal(got["gid"], np.sort(s.gid))
    pos = np.zeros_like(s.pos)
    pos[:, :3] = got["pos"][:, :3]  # gid g at row g (gids are 0..n-1)
    assert np.array_equal(got["gid"], np.arange(s.n))
    rows = np.random.default_rng(4).choice(s.n, 300, replace=False)
    ref = orc.lj_rows(pos, s.lo, s.hi, s.periodic, rc=2.5, r_min=0.8, rows=rows)
    err = orc.normalized_max_err(got["force"][rows, :3].astype(np.float64), ref["F"])
    assert err <= 1e-4, err
    for ctx in sim.m.values():
        ctx.close()


def test_torchrun_ipc_fused_refresh_two_processes(env):
    """The fused ghost refresh across PROCESSES (CUDA IPC mappings of the
    peer's position buffers, DistSim(peer=True)): two ranks on this GPU over
    gloo, 40 steps with rebuilds; the union of the owned states equals one
    context (tools/dist_peer_check.py asserts and prints "peer-ipc OK")."""
    import os
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(root, "tools", "dist_peer_check.py"), "24"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "peer-ipc OK" in r.stdout, r.stdout[-2000:]
