"""Multi-GPU groups through the C-ABI only (pm.h pm_create_dist_local,
pm_map, pm_ghost_get, pm_dist_run, pm_dist_thermo).

On one GPU the group's sub-domains live in this process: the
messages are device copies, or -- via_nccl -- NCCL point-to-point to the
process's own rank through a library-owned communicator, the code path a
multi-process group takes between GPUs.  Every test places the WHOLE global
system on member 0 and lets pm_map send each particle to its owner
(§3.4), so migration is exercised from the first call.
Checks: every particle owned exactly once, sampled rows' neighbour sets (as
gid sets, ghosts included) and forces against the fp64 oracle on the global
system, trajectory vs one context (rank-count independence, SURVEY §8(c)
"Multi-GPU")."""
import numpy as np
import pytest

from paper_1804_07598_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1804_07598_b200 import build, pm
    build.build()
    return pm


def make_group(pm, s, grid, via_nccl=False, place_on=0, stream=None):
    members = pm.create_dist_local(grid, via_nccl=via_nccl, stream=stream)
    for k, c in enumerate(members):
        c.set_domain(s.lo, s.hi, s.periodic)
        c.set_cutoff(2.5, 0.3)
        c.set_lj(1.0, 1.0, 1.0, 0.0)
        if k == place_on:
            c.place(s.pos, s.vel, s.gid)
        else:
            c.place(np.zeros((0, 4), np.float32), np.zeros((0, 4), np.float32),
                    np.zeros(0, np.int64))
    for c in members:
        c.map()
    for c in members:
        c.ghost_get()
    return members


def owned_union(pm, members):
    parts = [c.owned_state() for c in members]
    st = {k: np.concatenate([p[k] for p in parts]) for k in parts[0]}
    return pm.sorted_by_gid(st)


def forces(members, dt=0.005):
    for c in members:  # ghosts are current after pm_ghost_get
        c.dist_step(dt, 3)  # PM_PHASE_FORCES


def check_against_oracle(pm, members, s, nrow=120, seed=3):
    from oracle import oracle as orc
    inv = np.empty(int(s.gid.max()) + 1, np.int64)
    inv[s.gid] = np.arange(s.n)
    rv = np.float32(np.float32(2.5) + np.float32(0.3))
    rng = np.random.default_rng(seed)
    seen = 0
    for c in members:
        st = c.get_state()
        kind = c.get_kind()
        own = np.where((kind & pm.GHOST_BIT) == 0)[0]
        seen += own.size
        if own.size == 0:
            continue
        pick = rng.choice(own, min(nrow, own.size), replace=False)
        rp, col = c.get_verlet()
        rrp, rcols, _ = orc.verlet_rows(s.pos, s.lo, s.hi, s.periodic, rv,
                                        rows=inv[st["gid"][pick]], want_shift=False)
        for t, i in enumerate(pick):
            assert np.array_equal(np.sort(col[rp[i]:rp[i + 1]]),
                                  np.sort(s.gid[rcols[rrp[t]:rrp[t + 1]]])), f"row {i}"
        ref = orc.lj_rows(s.pos, s.lo, s.hi, s.periodic, rc=2.5, rows=inv[st["gid"][pick]])
        err = orc.normalized_max_err(st["force"][pick, :3].astype(np.float64), ref["F"])
        assert err <= 1e-4, err
    assert seen == s.n


@pytest.mark.parametrize("grid,via_nccl", [((2, 1, 1), False), ((2, 2, 2), False),
                                           ((2, 1, 1), True)])
def test_group_map_ghost_get_vs_oracle(env, grid, via_nccl):
    """cfg3-class blocks (BJ configs[2] recipe, 24^3 lattice per sub-domain):
    pm_map from one member, pm_ghost_get, forces; rows and forces vs the
    oracle on the global system."""
    pm = env
    s = inputs.cfg3_global(grid, m=24)
    members = make_group(pm, s, grid, via_nccl=via_nccl)
    info = [c.dist_info() for c in members]
    assert [i["sub_domain"] for i in info] == list(range(len(members)))
    forces(members)
    got = owned_union(pm, members)
    assert np.array_equal(got["gid"], np.sort(s.gid))  # every particle owned once
    check_against_oracle(pm, members, s)
    for c in members:
        c.close()


@pytest.mark.parametrize("grid,via_nccl,mode", [
    ((2, 1, 1), False, "fused"), ((2, 2, 2), False, "fused"), ((2, 1, 1), True, "fused"),
    ((2, 2, 2), False, "overlap"), ((2, 1, 1), True, "overlap"), ((2, 2, 1), False, "plain")])
def test_group_run_matches_single_context(env, grid, via_nccl, mode, monkeypatch):
    """40 NVE steps through pm_dist_run (rebuilds = pm_map + pm_ghost_get,
    per-step ghost refresh, MAX-reduced rebuild flag) against pm_step_vv on
    one context: positions, velocities and global thermo agree (fp32
    summation order only).  Refresh modes: fused into the sweep (default
    in-process), message exchange overlapped with the interior slices'
    forces (§3.6; opt-in, PM_GROUP_OVERLAP=1), plain message."""
    pm = env
    monkeypatch.setenv("PM_GROUP_FUSED", "1" if mode == "fused" else "0")
    monkeypatch.setenv("PM_GROUP_OVERLAP", "1" if mode == "overlap" else "0")
    s = inputs.lj_lattice_system(24, 24, 24, jitter_key=(52,), vel_key=(152,))
    ref = pm.Context()
    ref.set_domain(s.lo, s.hi, s.periodic)
    ref.set_cutoff(2.5, 0.3)
    ref.set_lj(1.0, 1.0, 1.0, 0.0)
    ref.place(s.pos, s.vel, s.gid)
    r = ref.step_vv(0.005, 40)
    rst = pm.sorted_by_gid(ref.get_state())
    members = make_group(pm, s, grid, via_nccl=via_nccl)
    out = [c.dist_run(0.005, 40) for c in members][-1]
    assert out["steps"] == 40 and out["rebuilds"] >= 2 and r["rebuilds"] >= 2
    got = owned_union(pm, members)
    assert np.array_equal(got["gid"], np.sort(s.gid))
    L = s.hi.astype(np.float64)
    d = got["pos"][:, :3].astype(np.float64) - rst["pos"][:, :3]
    d -= L * np.round(d / L)
    assert np.max(np.abs(d)) < 1e-3
    assert np.max(np.abs(got["vel"][:, :3] - rst["vel"][:, :3])) < 1e-2
    th = [c.dist_thermo() for c in members][-1]
    th_ref = ref.thermo()
    assert th["npairs"] == th_ref["npairs"]
    assert th["ke"] == pytest.approx(th_ref["ke"], rel=1e-4)
    assert th["pe_shift"] == pytest.approx(th_ref["pe_shift"], rel=1e-4)
    ref.close()
    for c in members:
        c.close()


@pytest.mark.parametrize("fused", ["1", "0"])
def test_group_batched_steps_equal_per_step_loop(env, fused, monkeypatch):
    """pm_dist_run in batches (PM_GROUP_BATCH: the rebuild flag reduced on the
    device into State::hold, held steps' kernels return at once, one host
    synchronisation per batch) gives bitwise the same trajectory as the
    per-step loop (batch 1): same arithmetic, same rebuild points, only the
    host synchronisations differ.  Batch 3 does not divide the rebuild
    interval, so held steps occur."""
    pm = env
    monkeypatch.setenv("PM_GROUP_FUSED", fused)
    s = inputs.lj_lattice_system(24, 24, 24, jitter_key=(54,), vel_key=(154,))
    res = []
    for batch in ("1", "3"):
        monkeypatch.setenv("PM_GROUP_BATCH", batch)
        members = make_group(pm, s, (2, 2, 1))
        out = [c.dist_run(0.005, 37) for c in members][-1]
        assert out["steps"] == 37 and out["rebuilds"] >= 2
        res.append((owned_union(pm, members), out["rebuilds"]))
        for c in members:
            c.close()
    (a, ra), (b, rb) = res
    assert ra == rb
    assert np.array_equal(a["gid"], b["gid"])
    assert np.array_equal(a["pos"], b["pos"]) and np.array_equal(a["vel"], b["vel"])


def test_group_empty_sub_domain(env):
    """A sub-domain with no particles: all particles in the lower
    half of x, grid (2,1,1) -- the upper member stays empty (no owned, only
    ghosts), builds, steps and flips in lock step; forces and a 20-step
    trajectory match one context."""
    pm = env
    s = inputs.lj_lattice_system(24, 12, 12, jitter_key=(53,), vel_key=(153,))
    keep = np.where(s.pos[:, 0] < 0.45 * s.hi[0])[0]
    s = s.subset(keep)
    members = make_group(pm, s, (2, 1, 1))
    counts = [c.count()["n_owned"] for c in members]
    assert counts[1] == 0 and counts[0] == s.n
    forces(members)
    check_against_oracle(pm, members, s)
    ref = pm.Context()
    ref.set_domain(s.lo, s.hi, s.periodic)
    ref.set_cutoff(2.5, 0.3)
    ref.set_lj(1.0, 1.0, 1.0, 0.0)
    ref.place(s.pos, s.vel, s.gid)
    ref.step_vv(0.005, 20)
    rst = pm.sorted_by_gid(ref.get_state())
    for c in members:
        c.dist_run(0.005, 20)
    got = owned_union(pm, members)
    assert np.array_equal(got["gid"], np.sort(s.gid))
    d = got["pos"][:, :3].astype(np.float64) - rst["pos"][:, :3]
    L = s.hi.astype(np.float64)
    d -= L * np.round(d / L)
    assert np.max(np.abs(d)) < 1e-3
    ref.close()
    for c in members:
        c.close()


def test_group_clustered_long_rows_vs_oracle(env):
    """Clustered input through the group API (BJ configs[4] recipe, 2 clusters
    of 32,768 at the config's local density, capped LJ r_min = 0.8): rows of
    thousands of entries (row-major slices, list relayout after the first
    overflowing build) on both sub-domains of (2,1,1); sampled rows over the
    length distribution and their capped forces against the oracle, then a
    short batched run keeps every particle."""
    pm = env
    from oracle import oracle as orc
    s = inputs.cfg5(n_clusters=2, per_cluster=32768)
    members = pm.create_dist_local((2, 1, 1))
    for k, c in enumerate(members):
        c.set_domain(s.lo, s.hi, s.periodic)
        c.set_cutoff(2.5, 0.3)
        c.set_lj(1.0, 1.0, 1.0, 0.8)
        if k == 0:
            c.place(s.pos, s.vel, s.gid)
        else:
            c.place(np.zeros((0, 4), np.float32), np.zeros((0, 4), np.float32),
                    np.zeros(0, np.int64))
    for c in members:
        c.map()
    for c in members:
        c.ghost_get()
    forces(members)
    inv = np.empty(int(s.gid.max()) + 1, np.int64)
    inv[s.gid] = np.arange(s.n)
    rv = np.float32(np.float32(2.5) + np.float32(0.3))
    longest = 0
    for c in members:
        st = c.get_state()
        own = np.where((c.get_kind() & pm.GHOST_BIT) == 0)[0]
        rp, col = c.get_verlet()
        lens = np.diff(rp)
        longest = max(longest, int(lens[own].max()))
        pick = own[np.argsort(lens[own])][np.linspace(0, own.size - 1, 24).astype(int)]
        rrp, rcols, _ = orc.verlet_rows(s.pos, s.lo, s.hi, s.periodic, rv,
                                        rows=inv[st["gid"][pick]], want_shift=False)
        for t, i in enumerate(pick):
            assert np.array_equal(np.sort(col[rp[i]:rp[i + 1]]),
                                  np.sort(s.gid[rcols[rrp[t]:rrp[t + 1]]])), f"row {i}"
        ref = orc.lj_rows(s.pos, s.lo, s.hi, s.periodic, rc=2.5, r_min=0.8,
                          rows=inv[st["gid"][pick]])
        err = orc.normalized_max_err(st["force"][pick, :3].astype(np.float64), ref["F"])
        assert err <= 1e-4, err
    assert longest > 1000
    for c in members:
        c.set_vlimit(0.15 / 0.005)
    out = [c.dist_run(0.005, 6) for c in members][-1]
    assert out["steps"] == 6
    got = owned_union(pm, members)
    assert np.array_equal(got["gid"], np.sort(s.gid))
    assert np.all(np.isfinite(got["pos"]))
    for c in members:
        c.close()


def test_group_call_order_errors(env):
    """Members must call the same collective: a member calling pm_ghost_get
    while another is inside pm_map is PM_E_STATE; a plain context is not a
    member."""
    pm = env
    s = inputs.cfg3_global((2, 1, 1), m=24)
    members = pm.create_dist_local((2, 1, 1))
    for k, c in enumerate(members):
        c.set_domain(s.lo, s.hi, s.periodic)
        c.set_cutoff(2.5, 0.3)
        c.set_lj(1.0, 1.0, 1.0, 0.0)
        c.place(s.pos if k == 0 else np.zeros((0, 4), np.float32))
    members[0].map()
    with pytest.raises(pm.PMError) as e:
        members[1].ghost_get()
    assert e.value.code == -2
    plain = pm.Context()
    with pytest.raises(pm.PMError) as e:
        pm.GroupMember.map(plain)
    assert e.value.code == -2
    plain.close()
    for c in members:
        c.close()


def test_bench_native_single_rank(env):
    """bench.py's N > 1 code path (dist.bench_native: pm_create_dist through a
    gloo-bootstrapped unique id, map, ghost_get, pm_dist_run with sweep
    profiling, e2e) at world size 1 under torchrun: one JSON line with the
    contract keys."""
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
    code = ("import sys; sys.path.insert(0, %r); import argparse, bench; "
            "from paper_1804_07598_b200 import dist; "
            "sys.exit(dist.bench_native(argparse.Namespace(steps=12, warmup=3)))" % root)
    script = os.path.join(root, "gpurun_out", "_bench_native_entry.py")
    os.makedirs(os.path.dirname(script), exist_ok=True)
    with open(script, "w") as f:
        f.write(code + "\n")
    env_ = dict(os.environ, PM_CFG3_BLOCK="32")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr", "127.0.0.1", "--master-port", str(port), script]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env_, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    b = json.loads(lines[0])
    assert b["n_gpus"] == 1 and b["config"]["n_particles"] == 32 ** 3
    assert b["value"] > 0 and b["e2e"]["value"] > 0 and b["roofline"]["frac"] > 0


def test_group_cfg3_full_size_222(env):
    """BJ configs[2] at full size on the 2x2x2 grid through the C-ABI group
    (8 sub-domains of one 128^3 block each = 16,777,216 particles on this
    GPU, placed on member 0 and distributed by pm_map): every particle owned
    once, sampled rows (gid sets, ghosts included) and forces of every
    sub-domain against the fp64 oracle on the global system, then 5 steps."""
    pm = env
    grid = (2, 2, 2)
    s = inputs.cfg3_global(grid)
    members = make_group(pm, s, grid)
    forces(members)
    check_against_oracle(pm, members, s, nrow=24, seed=8)
    out = [c.dist_run(0.005, 5) for c in members][-1]
    assert out["steps"] == 5
    assert sum(c.count()["n_owned"] for c in members) == s.n
    for c in members:
        c.close()
