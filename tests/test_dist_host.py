"""Host logic of the multi-GPU path on CPU: decomposition, neighbour/peer
maps, packing order and message segments, and the message protocol of
DistSim over a world-size-2 gloo process group (synthetic records stand in for
the CUDA pack/unpack kernels, which the GPU loopback test covers)."""
import os
import socket

import numpy as np
import pytest

from paper_1804_07598_b200.dist import DIRS, SELF, Decomp, DistSim, TorchTransport


def opposite(d):
    a = DIRS[d]
    return (-a[0] + 1) + 3 * (-a[1] + 1) + 9 * (-a[2] + 1)


@pytest.mark.parametrize("grid", [(1, 1, 1), (2, 1, 1), (2, 2, 1), (2, 2, 2), (3, 1, 1),
                                  (3, 3, 3), (4, 2, 1)])
def test_decomp_maps_are_consistent(grid):
    D = Decomp(grid)
    valid = D.valid_dirs()
    assert SELF not in valid
    n_dec = sum(1 for p in grid if p >= 2)
    assert len(valid) == 3 ** n_dec - 1
    for r in range(D.size):
        assert D.rank_of(D.coord(r)) == r
        order = D.send_order(r)
        assert sorted(order) == [d for d in range(27) if d != SELF]
        for d in valid:
            q = D.peer(r, d)
            assert q != r
            assert D.peer(q, opposite(d)) == r  # the way back
        # segments: contiguous, in peer order, sizes = sum of directions
        rng = np.random.default_rng(r)
        counts = np.zeros(27, np.int64)
        counts[valid] = rng.integers(0, 5, len(valid))
        seg = D.segments(r, counts)
        assert sorted(seg) == D.peers(r)
        off = 0
        for p in D.peers(r):
            o, n = seg[p]
            assert o == off
            assert n == sum(counts[d] for d in valid if D.peer(r, d) == p)
            off += n


class FakeCtx:
    """Stands in for pm.DistContext in the CPU protocol test: records are
    int64 (src rank, direction, k) triples packed as bytes."""

    def __init__(self, rank, D, rng_key):
        self.rank, self.D = rank, D
        self.counts = {}
        self.rng = np.random.default_rng(rng_key)
        self.arrived = {}

    def dist_plan(self, what, order):
        cnt = np.zeros(27, np.int64)
        for d in self.D.valid_dirs():
            cnt[d] = self.rng.integers(0, 4)
        self.counts[what] = (cnt, list(order))
        return cnt

    def dist_pack(self, what, buf):
        import torch
        cnt, order = self.counts[what]
        recs = [(self.rank, d, k) for d in order for k in range(int(cnt[d]))]
        if recs:
            arr = torch.tensor(recs, dtype=torch.int64).flatten()
            buf.view(torch.int64)[:arr.numel()] = arr

    def dist_unpack(self, what, buf, n):
        import torch
        self.arrived[what] = (buf.view(torch.int64)[:3 * n].reshape(-1, 3).tolist()
                              if n else [])

    def dist_finish(self):
        pass


def _worker(rank, world, port, grid, out):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    D = Decomp(grid)
    ctx = FakeCtx(rank, D, rng_key=(7, rank))
    sim = DistSim(D, {rank: ctx}, TorchTransport(device=None), device="cpu")
    from paper_1804_07598_b200 import pm
    import paper_1804_07598_b200.pm as pmm
    pmm.record_bytes = lambda what: 24  # 3 x int64 per synthetic record
    sim._message_round(pm.PM_MSG_GHOST)
    sent = {what: (c.tolist(), o) for what, (c, o) in ctx.counts.items()}
    out.put((rank, sent, ctx.arrived[pm.PM_MSG_GHOST], sim.ghost_recv[rank]))
    flag = sim._allreduce_max({rank: rank})
    out.put(("flag", rank, flag))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("grid", [(2, 1, 1), (1, 2, 1)])
def test_message_protocol_gloo_world2(grid):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, grid, q)) for r in range(2)]
    for p in procs:
        p.start()
    res, flags = {}, {}
    for _ in range(4):
        item = q.get(timeout=120)
        if item[0] == "flag":
            flags[item[1]] = item[2]
        else:
            res[item[0]] = item[1:]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert flags == {0: 1, 1: 1}
    D = Decomp(grid)
    from paper_1804_07598_b200 import pm
    for r in (0, 1):
        q_ = 1 - r
        sent_q, _, _ = res[q_]
        cnt_q, order_q = sent_q[pm.PM_MSG_GHOST]
        # what q sent to r, in q's packing order
        expect = [[q_, d, k] for d in order_q if d in D.valid_dirs() and D.peer(q_, d) == r
                  for k in range(cnt_q[d])]
        _, arrived, recv_counts = res[r]
        assert arrived == expect
        assert recv_counts[q_] == len(expect)


# ---------------------------------------------------------------- load balancing (NEXT-2)
def test_sar_stop_at_rise_examples():
    """SPEC.md:512-517 worked examples of the Stop-At-Rise rule W(n) =
    (C + sum delta)/n, re-balance at the first rise."""
    from paper_1804_07598_b200.dist import SAR
    s = SAR(10.0)
    out = []
    for times in ([1.0, 1.0], [2.0, 2.0]):  # delta 0, 0 -> W = 10, 5
        s.record(times)
        out.append(s.decide())
    assert out == [False, False]
    s.record([60.0, 0.0])  # delta 30 -> W = 40/3 > 5
    assert s.decide() is True
    s.record([100.0, 0.0])  # W rises again, but at most one True per reset
    assert s.decide() is False
    s.reset()
    assert not any((s.record([2.0, 0.0]), s.decide())[1] for _ in range(50))  # (10+n)/n falls


def test_weighted_cuts_balance_and_min_width():
    from paper_1804_07598_b200.dist import weighted_cuts
    rng = np.random.default_rng(3)
    x = rng.uniform(0, 100, 200000)
    c = weighted_cuts(x, np.ones_like(x), 4, 0.0, 100.0, 5.0)
    assert np.allclose(c, [25, 50, 75], atol=0.5)
    # a hotspot: 80% of the weight in [0, 20) pulls the cuts left
    w = np.where(x < 20, 16.0, 1.0)
    c = weighted_cuts(x, w, 4, 0.0, 100.0, 5.0)
    parts = [w[(x >= a) & (x < b)].sum() for a, b in zip([0, *c], [*c, 100])]
    assert max(parts) / np.mean(parts) < 1.02
    assert c[0] < 10 and np.all(np.diff(np.concatenate([[0], c, [100]])) >= 5.0)
    # the minimum width wins over the balance
    c = weighted_cuts(x, np.where(x < 2, 1e6, 1.0), 4, 0.0, 100.0, 5.0)
    assert np.all(np.diff(np.concatenate([[0], c, [100]])) >= 5.0 - 1e-9)


def test_owner_of_cuts_rule():
    """Ownership with cuts: slab = number of cuts <= x (the rule k_dist.cu
    applies); equal cuts reproduce the slabs of the uniform rule away from
    the rounding-sensitive faces."""
    from paper_1804_07598_b200 import dist, inputs
    s = inputs.random_box(5000, 40.0, (9,))
    D = dist.Decomp((2, 2, 1), cuts=(np.array([13.0], np.float32), np.array([30.0], np.float32),
                                     np.zeros(0, np.float32)))
    own = dist.owner_of(s, D)
    cx = (s.pos[:, 0] >= 13.0).astype(int)
    cy = (s.pos[:, 1] >= 30.0).astype(int)
    assert np.array_equal(own, cx + 2 * cy)


def _hybrid_worker(rank, world, port, grid, assign, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1804_07598_b200.dist import HybridTransport
    import paper_1804_07598_b200.pm as pmm
    pmm.record_bytes = lambda what: 24  # 3 x int64 per synthetic record
    D = Decomp(grid)
    tr = HybridTransport(assign, rank, TorchTransport(device=None))
    ctxs = {sd: FakeCtx(sd, D, rng_key=(11, sd)) for sd in tr.local}
    sim = DistSim(D, ctxs, tr, device="cpu")
    sim._message_round(pmm.PM_MSG_GHOST)
    for sd, ctx in ctxs.items():
        out.put((sd, {w: (c.tolist(), o) for w, (c, o) in ctx.counts.items()},
                 ctx.arrived[pmm.PM_MSG_GHOST]))
    out.put(("flag", rank, sim._allreduce_max({sd: sd for sd in ctxs})))
    dist.destroy_process_group()


def test_hybrid_transport_over_decomposition_gloo_world2():
    """Over-decomposition (NEXT-2): 8 sub-domains of a 2x2x2 grid on 2
    processes with a mixed assignment; every sub-domain receives exactly the
    records its peers packed for it, in peer order, whether the peer is local
    (device copy) or remote (one concatenated transfer per process pair)."""
    import torch.multiprocessing as mp
    grid, assign = (2, 2, 2), [0, 1, 1, 0, 1, 0, 0, 1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_hybrid_worker, args=(r, 2, port, grid, assign, q))
             for r in range(2)]
    for p in procs:
        p.start()
    res, flags = {}, {}
    for _ in range(10):
        item = q.get(timeout=120)
        if item[0] == "flag":
            flags[item[1]] = item[2]
        else:
            res[item[0]] = item[1:]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert flags == {0: 7, 1: 7}
    D = Decomp(grid)
    from paper_1804_07598_b200 import pm
    for r in range(8):
        expect = []
        for q_ in D.peers(r):  # arrivals are concatenated in peer order
            cnt_q, order_q = res[q_][0][pm.PM_MSG_GHOST]
            expect += [[q_, d, k] for d in order_q if d in D.valid_dirs() and D.peer(q_, d) == r
                       for k in range(cnt_q[d])]
        assert res[r][1] == expect


class FakeSPHCtx(FakeCtx):
    """FakeCtx plus the SPH stepping calls: a rank-dependent local step bound,
    and a record of the bound each update was given."""

    def __init__(self, rank, D, rng_key):
        super().__init__(rank, D, rng_key)
        self.bounds_seen = []
        self.step = 0

    def dist_sph_init(self):
        pass

    def dist_sph_rates(self):
        self.step += 1
        return float(np.float32(1e-4 * (1.0 + 0.5 * ((self.rank + self.step) % 3))))

    def dist_sph_update(self, bound, cfl, every):
        self.bounds_seen.append(bound)
        return int(self.rank == 1 and self.step == 2)  # one rank asks for a rebuild once

    def refresh_pack(self, buf, pv=False):
        assert pv
        import torch
        n = buf.numel() // 32 if buf is not None else 0
        if n:
            buf.view(torch.float32)[:] = float(self.rank)

    def refresh_unpack(self, buf, pv=False):
        import torch
        self.refreshed = [] if buf is None else sorted(set(buf.view(torch.float32).tolist()))


def _sph_worker(rank, world, port, grid, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1804_07598_b200.pm as pmm
    pmm.record_bytes = lambda what: 24
    D = Decomp(grid)
    ctx = FakeSPHCtx(rank, D, rng_key=(21, rank))
    sim = DistSim(D, {rank: ctx}, TorchTransport(device=None), device="cpu")
    sim.sph_start()
    reb, t = sim.sph_run(4, cfl=0.5, every=10)
    out.put((rank, ctx.bounds_seen, reb, t, ctx.refreshed))
    dist.destroy_process_group()


def test_sph_stepping_protocol_gloo_world2():
    """DistSim.sph_run over world-size-2 gloo (NEXT-3 multi-GPU SPH): every
    update gets the global minimum of the ranks' fp32 step bounds (exact
    MIN all-reduce), a rebuild asked by one rank happens on both, and the
    ghost refresh moves 32-byte records from the peer."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sph_worker, args=(r, 2, port, (2, 1, 1), q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        item = q.get(timeout=120)
        res[item[0]] = item[1:]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    expect = [float(np.float32(1e-4 * (1.0 + 0.5 * min((r + s) % 3 for r in (0, 1)))))
              for s in range(1, 5)]
    for r in (0, 1):
        bounds, reb, t, refreshed = res[r]
        assert bounds == expect
        assert reb == 1
        assert t == pytest.approx(0.5 * sum(expect))
        assert refreshed == [float(1 - r)]


class FakeDEMCtx(FakeCtx):
    """FakeCtx that also packs the MIGRATE_HIST records of a DEM migration:
    (1000 + rank, direction, k) for the k-th leaver towards each direction."""

    def dist_pack(self, what, buf):
        import torch
        from paper_1804_07598_b200 import pm
        if what == pm.PM_MSG_MIGRATE_HIST:
            cnt, order = self.counts[pm.PM_MSG_MIGRATE]
            recs = [(1000 + self.rank, d, k) for d in order for k in range(int(cnt[d]))]
            if recs:
                arr = torch.tensor(recs, dtype=torch.int64).flatten()
                buf.view(torch.int64)[:arr.numel()] = arr
            return
        super().dist_pack(what, buf)


def _dem_worker(rank, world, port, grid, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1804_07598_b200.pm as pmm
    pmm.record_bytes = lambda what: 24
    D = Decomp(grid)
    ctx = FakeDEMCtx(rank, D, rng_key=(31, rank))
    sim = DistSim(D, {rank: ctx}, TorchTransport(device=None), device="cpu")
    sim.dem = True
    sim._message_round(pmm.PM_MSG_MIGRATE)
    out.put((rank, ctx.arrived[pmm.PM_MSG_MIGRATE], ctx.arrived[pmm.PM_MSG_MIGRATE_HIST]))
    dist.destroy_process_group()


def test_dem_migration_histories_ride_with_grains_gloo_world2():
    """A decomposed DEM migration round over world-size-2 gloo: the contact
    history records (PM_MSG_MIGRATE_HIST) use the MIGRATE counts and
    segments, so the k-th history record that arrives belongs to the k-th
    grain that arrives."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dem_worker, args=(r, 2, port, (2, 1, 1), q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        item = q.get(timeout=120)
        res[item[0]] = item[1:]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    total = 0
    for r in (0, 1):
        mig, hist = res[r]
        assert len(mig) == len(hist)
        assert [[a - 1000, d, k] for a, d, k in hist] == mig
        total += len(mig)
    assert total > 0


class FakePutCtx(FakeCtx):
    """Packs one 16-byte record per arrived ghost: (rank, arrival index)."""

    def ghost_put_pack(self, buf):
        import torch
        n = buf.numel() // 16 if buf is not None else 0
        if n:
            v = buf.view(torch.int64).view(-1, 2)
            v[:, 0] = self.rank
            v[:, 1] = torch.arange(n)

    def ghost_put_unpack(self, buf):
        import torch
        self.put = [] if buf is None else buf.view(torch.int64).view(-1, 2).tolist()


def _put_worker(rank, world, port, grid, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1804_07598_b200.pm as pmm
    pmm.record_bytes = lambda what: 24
    D = Decomp(grid)
    ctx = FakePutCtx(rank, D, rng_key=(41, rank))
    sim = DistSim(D, {rank: ctx}, TorchTransport(device=None), device="cpu")
    sim._message_round(pmm.PM_MSG_GHOST)
    sim._ghost_put()
    sent = ctx.counts[pmm.PM_MSG_GHOST][0].tolist()
    out.put((rank, sent, sim.ghost_recv[rank], ctx.put))
    dist.destroy_process_group()


def test_ghost_put_reverses_the_ghost_round_gloo_world2():
    """ghost_put (NEXT-1 half lists across sub-domains) over world-size-2
    gloo: each arrived ghost's share goes back to the rank that sent the
    ghost, landing in that rank's send order."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_put_worker, args=(r, 2, port, (2, 1, 1), q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        item = q.get(timeout=120)
        res[item[0]] = item[1:]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in (0, 1):
        sent, _, put = res[r]
        other = 1 - r
        n_sent = sum(sent)  # records r packed as ghosts for the other rank
        assert res[other][1][r] == n_sent  # the other rank received them
        assert put == [[other, k] for k in range(n_sent)]


def test_histogram_cuts_match_gathered_quantiles_and_are_rank_independent():
    """NEXT-2 without a global gather: cuts from summed
    per-rank histograms equal (to one bin) the weighted quantiles of the
    gathered particles, do not depend on how the particles are split over
    ranks, and keep slabs >= 2 r_v."""
    from paper_1804_07598_b200.dist import histogram_cuts, weighted_cuts
    rng = np.random.default_rng(5)
    L = 120.0
    x = np.concatenate([rng.normal(30, 6, (40000, 3)), rng.uniform(0, L, (20000, 3))]) % L
    w = rng.uniform(20, 80, x.shape[0])
    grid = (4, 2, 1)
    lo, hi = np.zeros(3), np.full(3, L)
    parts = np.array_split(rng.permutation(x.shape[0]), 3)  # three "ranks"
    hs = []

    def collect(h):
        hs.append(h)
        return h
    # every rank's histogram, then their sum (what an all-reduce would return)
    for p_ in parts:
        histogram_cuts(grid, x[p_], w[p_], lo, hi, 2.8, collect, bins=4096)
    tot = sum(hs)
    c_split = histogram_cuts(grid, x[parts[0]], w[parts[0]], lo, hi, 2.8, lambda h: tot,
                             bins=4096)
    c_all = histogram_cuts(grid, x, w, lo, hi, 2.8, lambda h: h, bins=4096)
    for d in range(3):
        assert np.array_equal(c_split[d], c_all[d])
        if grid[d] > 1:
            q = weighted_cuts(x[:, d], w, grid[d], 0.0, L, 2.8 * 2 * (1 + 1e-5))
            assert np.all(np.abs(q - c_all[d]) <= L / 4096 + 1e-3)
            edges = np.concatenate([[0.0], c_all[d], [L]])
            assert np.all(np.diff(edges) >= 5.6)
        else:
            assert c_all[d].size == 0
