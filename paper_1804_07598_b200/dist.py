"""Multi-GPU orchestration of the decomposed hot path.

The periodic box is split into px x py x pz cuboids, one per rank (GPU); each
rank's pm_ctx owns one cuboid (pm_set_decomposition).  PAPER.md:62 (§3.1):
sub-domains extended by a ghost layer of interaction width; PAPER.md:112-118
(§3.4): map() migrates particles that left a sub-domain to the neighbour that
owns them and ghost_get() fills the ghost layers (here with positions only
between rebuilds, PAPER.md:118 and Listing 4.1 ghost_get<>()).

All particle work (selection, packing, unpacking, sorting, lists, forces,
integration) runs in libpm.so kernels.  This module only decides who talks to
whom, moves message bytes with a Transport, and sequences the phases:

  rebuild:  plan/pack MIGRATE -> exchange -> unpack; plan/pack GHOST ->
            exchange -> unpack; finish (cells, lists, refresh maps)
  step:     [rebuild if any rank's particle moved > skin/2, else ghost
            refresh] -> force + fused kick/drift -> global flag (MAX)

Transports: TorchTransport (torch.distributed: NCCL between GPUs, gloo on
CPU for the host-logic tests) and LoopbackTransport (several sub-domains in
one process on one GPU -- a test stand-in for NVLink that exercises exactly
the same kernels and message layout).
"""
from __future__ import annotations

import itertools
import json
import os
import time
from dataclasses import dataclass

import numpy as np

# direction index d = (ax+1) + 3 (ay+1) + 9 (az+1); 13 = self
DIRS = [(ax, ay, az) for az in (-1, 0, 1) for ay in (-1, 0, 1) for ax in (-1, 0, 1)]
SELF = 13


def dir_index(a):
    return (a[0] + 1) + 3 * (a[1] + 1) + 9 * (a[2] + 1)


@dataclass
class Decomp:
    """px x py x pz cuboids; rank = cx + px (cy + py cz).  cuts: None (equal
    cuboids) or, per axis, the grid[d]-1 interior cut positions of a
    load-balanced tensor-product decomposition (pm_set_decomposition_cuts)."""

    grid: tuple
    cuts: tuple = None

    @property
    def size(self):
        return self.grid[0] * self.grid[1] * self.grid[2]

    def coord(self, rank):
        px, py, _ = self.grid
        return (rank % px, (rank // px) % py, rank // (px * py))

    def rank_of(self, c):
        px, py, pz = self.grid
        return (c[0] % px) + px * ((c[1] % py) + py * (c[2] % pz))

    def valid_dirs(self):
        """Directions that exist: no component along an undecomposed axis
        (computed once per grid: the rebuild path asks for it per message)."""
        key = tuple(self.grid)
        cache = self.__dict__.setdefault("_vd", {})
        if key not in cache:
            cache[key] = [d for d, a in enumerate(DIRS)
                          if d != SELF and all(a[k] == 0 or self.grid[k] >= 2 for k in range(3))]
        return cache[key]

    def peer(self, rank, d):
        c = self.coord(rank)
        a = DIRS[d]
        return self.rank_of(tuple(c[k] + a[k] for k in range(3)))

    def peers(self, rank):
        return sorted({self.peer(rank, d) for d in self.valid_dirs()})

    def send_order(self, rank):
        """Packing order of the 26 directions: grouped by peer (ascending),
        then by direction index; non-existent directions last (always empty)."""
        key = (tuple(self.grid), rank)
        cache = self.__dict__.setdefault("_so", {})
        if key not in cache:
            v = self.valid_dirs()
            order = sorted(v, key=lambda d: (self.peer(rank, d), d))
            order += [d for d in range(27) if d != SELF and d not in v]
            cache[key] = order
        return list(cache[key])

    def segments(self, rank, counts):
        """Per peer: (first record, number of records) of its segment in the
        buffer packed in send_order (counts = per-direction records)."""
        seg, off = {}, 0
        valid = set(self.valid_dirs())
        for d in self.send_order(rank):
            if d not in valid:
                assert counts[d] == 0
                continue
            p = self.peer(rank, d)
            if p not in seg:
                seg[p] = [off, 0]
            seg[p][1] += int(counts[d])
            off += int(counts[d])
        for p in self.peers(rank):
            seg.setdefault(p, [off, 0])
        return {p: tuple(v) for p, v in seg.items()}


# ---------------------------------------------------------------- transports
class TorchTransport:
    """torch.distributed point-to-point (NCCL on GPUs; gloo on CPU)."""

    def __init__(self, device=None, stage_host=False):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.device = device
        # gloo between ranks that share a GPU (tests): device buffers go through
        # host copies; the library kernels never wait on another rank
        self.stage_host = stage_host

    def exchange(self, sends, recvs):
        """sends/recvs: {peer: tensor} (uint8 or int64); zero-size skipped."""
        if self.stage_host:
            hs = {p: t.cpu() for p, t in sends.items()}
            hr = {p: self.torch.empty(t.shape, dtype=t.dtype) for p, t in recvs.items()}
            self._exchange(hs, hr)
            for p, t in recvs.items():
                if t.numel() > 0:
                    t.copy_(hr[p])
            return
        self._exchange(sends, recvs)

    def _exchange(self, sends, recvs):
        ops = []
        P2P, dist = self.dist.P2POp, self.dist
        for p in sorted(set(sends) | set(recvs)):
            if p in sends and sends[p].numel() > 0:
                ops.append(P2P(dist.isend, sends[p], p))
            if p in recvs and recvs[p].numel() > 0:
                ops.append(P2P(dist.irecv, recvs[p], p))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()

    def exchange_counts(self, counts):
        """counts: {peer: int} -> {peer: int received}."""
        t = self.torch
        dev = self.device if self.device is not None else "cpu"
        s = {p: t.tensor([int(c)], dtype=t.int64, device=dev) for p, c in counts.items()}
        r = {p: t.zeros(1, dtype=t.int64, device=dev) for p in counts}
        self.exchange(s, r)
        return {p: int(v.item()) for p, v in r.items()}

    def allreduce_max(self, x):
        t = self.torch
        dev = self.device if self.device is not None else "cpu"
        v = t.tensor([int(x)], dtype=t.int64, device=dev)
        self.dist.all_reduce(v, op=self.dist.ReduceOp.MAX)
        return int(v.item())

    def allreduce_sum(self, arr):
        t = self.torch
        dev = self.device if self.device is not None else "cpu"
        v = t.tensor(np.asarray(arr, np.float64), device=dev)
        self.dist.all_reduce(v)
        return v.cpu().numpy()

    def allreduce_min_f32(self, x):
        """Exact global minimum of one fp32 value (the SPH step bound)."""
        t = self.torch
        dev = self.device if self.device is not None else "cpu"
        v = t.tensor([x], dtype=t.float32, device=dev)
        self.dist.all_reduce(v, op=self.dist.ReduceOp.MIN)
        return float(v.item())


class LoopbackTransport:
    """All ranks live in this process (lock-step): a message from rank r to
    peer q is a device-to-device copy.  Used to run P sub-domains on one GPU."""

    def __init__(self, members):
        self.members = members  # rank -> object with .rank

    def exchange_all(self, sends, recvs):
        """sends[r][q] -> recvs[q][r] (tensors of equal size)."""
        for r, per in sends.items():
            for q, buf in per.items():
                if buf.numel() > 0:
                    recvs[q][r].copy_(buf)

    def exchange_counts_all(self, counts):
        return {q: {r: counts[r][q] for r in counts if q in counts[r]} for q in counts}


# ---------------------------------------------------------------- simulation
class HybridTransport:
    """Over-decomposition (the paper assigns sub-sub-domains
    to processors): several sub-domains per process.
    Messages between local sub-domains are device copies; all messages from
    this process to one remote process travel as ONE point-to-point transfer
    (torch.distributed, NCCL on GPUs), concatenated in (sender, receiver)
    sub-domain order, and are split the same way on arrival.

    assign[sd] = rank of sub-domain sd; local = the sub-domains of this
    process; torch_tr = TorchTransport (None: every sub-domain is local)."""

    def __init__(self, assign, my_rank, torch_tr=None):
        self.assign = np.asarray(assign, np.int64)
        self.rank = int(my_rank)
        self.tr = torch_tr
        self.local = [int(s) for s in np.where(self.assign == self.rank)[0]]

    def exchange_counts_all(self, counts):
        """counts[r][q] (r local) -> {q local: {r: n}} over all senders r."""
        S = self.assign.size
        M = np.zeros((S, S), np.int64)
        for r, per in counts.items():
            for q, n in per.items():
                M[r, q] = int(n)
        if self.tr is not None:
            M = np.rint(self.tr.allreduce_sum(M.astype(np.float64).reshape(-1))).astype(
                np.int64).reshape(S, S)
        return {q: {r: int(M[r, q]) for r in range(S) if r != q} for q in self.local}

    def exchange_all(self, sends, recvs):
        """sends[r][q] (r local) -> recvs[q][r] (q local), uint8 tensors."""
        import torch
        remote_out, remote_in = {}, {}
        for r in sorted(sends):
            for q in sorted(sends[r]):
                buf = sends[r][q]
                if buf.numel() == 0:
                    continue
                R = int(self.assign[q])
                if R == self.rank:
                    recvs[q][r].copy_(buf)
                else:
                    remote_out.setdefault(R, []).append(buf)
        # incoming pieces in the senders' (sender, receiver) order
        pairs = sorted((r, q) for q in recvs for r in recvs[q]
                       if int(self.assign[r]) != self.rank and recvs[q][r].numel() > 0)
        for r, q in pairs:
            remote_in.setdefault(int(self.assign[r]), []).append(recvs[q][r])
        if not remote_out and not remote_in:
            return
        if self.tr is None:
            raise RuntimeError("HybridTransport: remote sub-domain without a process group")
        outs = {R: torch.cat(v) for R, v in remote_out.items()}
        ins = {R: torch.empty(sum(t.numel() for t in v), dtype=torch.uint8, device=v[0].device)
               for R, v in remote_in.items()}
        self.tr.exchange(outs, ins)
        for R, v in remote_in.items():
            off = 0
            for t in v:
                t.copy_(ins[R][off:off + t.numel()])
                off += t.numel()

    def allreduce_max(self, x):
        return x if self.tr is None else self.tr.allreduce_max(x)

    def allreduce_min_f32(self, x):
        return x if self.tr is None else self.tr.allreduce_min_f32(x)

    def allreduce_sum(self, arr):
        return np.asarray(arr, np.float64) if self.tr is None else self.tr.allreduce_sum(arr)


def lpt_assign(work, nranks):
    """Longest-processing-time greedy assignment of sub-domains to ranks
    (heaviest first onto the least loaded rank; deterministic)."""
    load = np.zeros(nranks)
    assign = np.zeros(len(work), np.int64)
    for i in np.argsort(-np.asarray(work, np.float64), kind="stable"):
        r = int(np.argmin(load))
        assign[i] = r
        load[r] += work[i]
    return assign


class DistSim:
    """Lock-step driver for one or more local sub-domains.

    members: {rank: pm.DistContext}; transport: TorchTransport (one local
    member per process) or LoopbackTransport (all members local)."""

    def __init__(self, decomp: Decomp, members: dict, transport, dt=0.005, device="cuda",
                 stream=None, peer=None, newton=False):
        import contextlib
        import torch
        self.torch = torch
        self.device = device
        # all library work, buffer copies and NCCL calls are ordered on ONE
        # stream: the members must have been created on it (make_member)
        self.stream = stream
        self._ctxmgr = (lambda: torch.cuda.stream(stream)) if stream is not None \
            else contextlib.nullcontext
        self.D = decomp
        self.m = members
        self.tr = transport
        self.dt = dt
        self.loop = isinstance(transport, LoopbackTransport)
        self.multi = hasattr(transport, "exchange_all")  # all local members at once
        self.dem = False      # DEM runs: migrations carry contact histories
        self.prof = None      # list: (start, end) CUDA events around each step's sweep
        # fused ghost refresh: the sweep stores new positions straight into
        # the peers' ghost slots (loopback: same-process pointers; processes:
        # CUDA IPC).  Opt-in: PM_DIST_PEER=1 or peer=True.
        self.peer = bool(int(os.environ.get("PM_DIST_PEER", "0"))) if peer is None else peer
        self._ipc_key = None
        # half (Newton) lists across sub-domains: pairs once, the ghosts'
        # force shares go back to their owners every step (ghost_put)
        self.newton = newton
        if newton and self.peer:  # the half-list integrator has no fused stores
            raise ValueError("DistSim: the fused ghost refresh needs full lists (newton=False)")
        if newton:
            for ctx in members.values():
                ctx.set_newton(True)
        self.sar = None       # SAR trigger: runtime re-balancing (enable_rebalance)
        self.rebalances = 0
        self.ghost_seg = {}   # rank -> {peer: (off, n)} of the last ghost plan (send side)
        self.ghost_recv = {}  # rank -> {peer: n} received ghosts
        self.rebuilds = 0
        self._bufs = {}

    # ---- helpers
    def _buf(self, key, nbytes):
        t = self.torch
        b = self._bufs.get(key)
        if b is None or b.numel() < nbytes:
            b = t.empty(max(int(nbytes * 1.25), 64), dtype=t.uint8, device=self.device)
            self._bufs[key] = b
        return b[:nbytes]

    def _exchange(self, sends, recvs):
        if self.multi:
            self.tr.exchange_all(sends, recvs)
        else:
            (r,) = list(self.m)
            self.tr.exchange(sends[r], recvs[r])

    def _exchange_counts(self, counts):
        if self.multi:
            return self.tr.exchange_counts_all(counts)
        (r,) = list(self.m)
        return {r: self.tr.exchange_counts(counts[r])}

    # ---- runtime re-balancing (§3.5)
    def enable_rebalance(self, cost_ms=1.0, bins=4096):
        """Stop-At-Rise re-balancing inside run(): every step records the
        per-rank step times (CUDA events around each rank's sweep); when SAR
        fires, the cuts are recomputed from all-reduced pair-work histograms
        (histogram_cuts), every member gets them (pm_set_decomposition_cuts)
        and the next step migrates (map) and rebuilds the ghosts.  cost_ms:
        the first estimate of a re-balance (then the measured one)."""
        self.sar = SAR(cost_ms)
        self._bins = bins

    def _allsum(self, arr):
        arr = np.asarray(arr, np.float64)
        if self.loop:
            return arr
        return self.tr.allreduce_sum(arr)

    def _rank_times(self, local):
        """{rank: ms} of the local members -> the vector over all ranks."""
        v = np.zeros(self.D.size)
        for r, t in local.items():
            v[r] = t
        return self._allsum(v)

    def rebalance(self):
        """New load-balanced cuts from the current particles (no gather: each
        member contributes a histogram of its owned coordinates weighted by
        its Verlet row lengths), applied to every member; the caller rebuilds
        (map + ghost_get).  Returns the new Decomp."""
        from . import pm
        pos, w = [], []
        for ctx in self.m.values():
            st = ctx.get_state()
            rp, _ = ctx.get_verlet(cols=False)
            own = (ctx.get_kind() & pm.GHOST_BIT) == 0
            pos.append(st["pos"][own, :3])
            w.append(np.diff(rp)[own] + 1.0)  # pair work (+1: the particle itself)
        ctx0 = next(iter(self.m.values()))
        lo, hi = ctx0._box
        rv = ctx0._rv
        cuts = histogram_cuts(self.D.grid, np.concatenate(pos), np.concatenate(w), lo, hi, rv,
                              self._allsum, self._bins)
        D = Decomp(self.D.grid, cuts)
        for r, ctx in self.m.items():
            ctx.set_decomposition_cuts(D.grid, D.coord(r), cuts)
        self.D = D
        self.rebalances += 1
        return D

    def _allreduce_max(self, vals):
        v = max(vals.values())
        return v if self.loop else self.tr.allreduce_max(v)

    def _message_round(self, what):
        """plan -> pack -> counts -> exchange -> unpack for MIGRATE / GHOST."""
        from . import pm
        rb = pm.record_bytes(what)
        dem = self.dem and what == pm.PM_MSG_MIGRATE
        hb = pm.record_bytes(pm.PM_MSG_MIGRATE_HIST) if dem else 0
        hist_sends = {} if dem else None
        sends, seg, counts = {}, {}, {}
        for r, ctx in self.m.items():
            cnt = ctx.dist_plan(what, self.D.send_order(r))
            seg[r] = self.D.segments(r, cnt)
            nsend = sum(n for _, n in seg[r].values())
            if dem:  # before the MIGRATE pack removes the leavers
                hbuf = self._buf(("hsend", r), nsend * hb)
                ctx.dist_pack(pm.PM_MSG_MIGRATE_HIST, hbuf if nsend else None)
                hist_sends[r] = {p: hbuf[o * hb:(o + n) * hb] for p, (o, n) in seg[r].items()}
            buf = self._buf(("send", what, r), nsend * rb)
            ctx.dist_pack(what, buf if nsend else None)
            sends[r] = {p: buf[o * rb:(o + n) * rb] for p, (o, n) in seg[r].items()}
            counts[r] = {p: n for p, (o, n) in seg[r].items()}
        recv_counts = self._exchange_counts(counts)

        def recv_bufs(kind, rsz):
            recvs, rbufs = {}, {}
            for r in self.m:
                peers = self.D.peers(r)
                tot = sum(recv_counts[r][p] for p in peers)
                buf = self._buf(("recv", kind, r), tot * rsz)
                rbufs[r] = (buf, tot)
                off, recvs[r] = 0, {}
                for p in peers:  # arrivals concatenated in peer order
                    n = recv_counts[r][p]
                    recvs[r][p] = buf[off * rsz:(off + n) * rsz]
                    off += n
            return recvs, rbufs

        recvs, rbufs = recv_bufs(what, rb)
        self._exchange(sends, recvs)
        for r, ctx in self.m.items():
            buf, tot = rbufs[r]
            ctx.dist_unpack(what, buf if tot else None, tot)
        if hist_sends is not None:  # DEM: the leavers' contact histories, same counts
            recvs, rbufs = recv_bufs(pm.PM_MSG_MIGRATE_HIST, hb)
            self._exchange(hist_sends, recvs)
            for r, ctx in self.m.items():
                buf, tot = rbufs[r]
                ctx.dist_unpack(pm.PM_MSG_MIGRATE_HIST, buf if tot else None, tot)
        if what == pm.PM_MSG_GHOST:
            self.ghost_seg = seg
            self.ghost_recv = recv_counts

    def rebuild(self):
        with self._ctxmgr():
            self._rebuild()

    def _rebuild(self):
        from . import pm
        self._message_round(pm.PM_MSG_MIGRATE)
        self._message_round(pm.PM_MSG_GHOST)
        for ctx in self.m.values():
            ctx.dist_finish()
        if self.peer:
            self._peer_setup()
        self.rebuilds += 1

    def _recv_off(self, q, r):
        """First record of sender r among receiver q's ghost arrivals."""
        off = 0
        for p in self.D.peers(q):
            if p == r:
                return off
            off += self.ghost_recv[q][p]
        raise KeyError((q, r))

    def _peer_setup(self):
        """Fused ghost refresh tables after a rebuild: per ghost send entry its
        peer index and the receiver's ghost slot; the peers' position buffers."""
        t = self.torch
        slots = {}
        for r, ctx in self.m.items():
            ng = sum(self.ghost_recv[r].values())
            buf = t.empty(max(ng, 1), dtype=t.int32, device=self.device)
            ctx.ghost_slots(buf if ng else None)
            slots[r] = buf
        if self.loop:
            bufs = {r: ctx.pos_buffers() for r, ctx in self.m.items()}
            for r, ctx in self.m.items():
                peers = self.D.peers(r)
                nsend = sum(n for _, n in self.ghost_seg[r].values())
                dp = t.empty(max(nsend, 1), dtype=t.int32, device=self.device)
                ds = t.empty(max(nsend, 1), dtype=t.int32, device=self.device)
                for k, q in enumerate(peers):
                    o, n = self.ghost_seg[r][q]
                    if n:
                        ro = self._recv_off(q, r)
                        dp[o:o + n] = k
                        ds[o:o + n] = slots[q][ro:ro + n]
                ctx.peer_setup([bufs[q] for q in peers], dp, ds)
            return
        # processes: the receivers return their slot slices (reverse of the
        # ghost round), position buffers through CUDA IPC
        (r, ctx), = self.m.items()
        peers = self.D.peers(r)
        sends = {q: slots[r][self._recv_off(r, q):self._recv_off(r, q) + self.ghost_recv[r][q]]
                 for q in peers}
        nsend = sum(n for _, n in self.ghost_seg[r].values())
        ds = t.empty(max(nsend, 1), dtype=t.int32, device=self.device)
        dp = t.empty(max(nsend, 1), dtype=t.int32, device=self.device)
        recvs = {q: ds[o:o + n] for q, (o, n) in self.ghost_seg[r].items()}
        self.tr.exchange(sends, recvs)
        for k, q in enumerate(peers):
            o, n = self.ghost_seg[r][q]
            dp[o:o + n] = k
        import torch.distributed as tdist
        hs = [None] * tdist.get_world_size()
        tdist.all_gather_object(hs, ctx.ipc_handles())  # any rank may have reallocated
        if self._ipc_key != hs:
            ctx.ipc_close_all()
            self._peer_bufs = [ctx.ipc_open(hs[q]) for q in peers]
            self._ipc_key = hs
        ctx.peer_setup(self._peer_bufs, dp, ds)

    def refresh(self):
        with self._ctxmgr():
            self._refresh()

    def _refresh(self, pv=False):
        """Ghost refresh with the last ghost plan's layout: positions only
        (16 B per ghost), positions and velocities (pv, 32 B: SPH runs), or
        also angular velocities (pv="pvw", 48 B: DEM runs)."""
        rsz = {False: 16, True: 32, "pv": 32, "pvw": 48}[pv]
        sends, recvs = {}, {}
        for r, ctx in self.m.items():
            nsend = sum(n for _, n in self.ghost_seg[r].values())
            buf = self._buf(("rsend", r), nsend * rsz)
            ctx.refresh_pack(buf if nsend else None, pv=pv)
            sends[r] = {p: buf[o * rsz:(o + n) * rsz] for p, (o, n) in self.ghost_seg[r].items()}
        rb = {}
        for r in self.m:
            peers = self.D.peers(r)
            tot = sum(self.ghost_recv[r][p] for p in peers)
            buf = self._buf(("rrecv", r), tot * rsz)
            rb[r] = (buf, tot)
            off, recvs[r] = 0, {}
            for p in peers:
                n = self.ghost_recv[r][p]
                recvs[r][p] = buf[off * rsz:(off + n) * rsz]
                off += n
        self._exchange(sends, recvs)
        for r, ctx in self.m.items():
            buf, tot = rb[r]
            ctx.refresh_unpack(buf if tot else None, pv=pv)

    def start(self):
        """After pm_place on every member: first decomposition + forces."""
        from . import pm
        with self._ctxmgr():
            self._rebuild()
            if self.newton:
                self._newton_forces()
            else:
                for ctx in self.m.values():
                    ctx.dist_step(self.dt, pm.PM_PHASE_FORCES)

    def _newton_forces(self):
        from . import pm
        for ctx in self.m.values():
            ctx.dist_step(self.dt, pm.PM_PHASE_NEWTON_FORCES)
        self._ghost_put()

    def _ghost_put(self):
        """The force shares on the ghost copies back to their owners (16 B per
        ghost): the ghost round reversed -- a receiver's arrivals per peer go
        back to that peer, which adds them in its send order."""
        sends, recvs, rb = {}, {}, {}
        for r, ctx in self.m.items():
            ng = sum(self.ghost_recv[r].values())
            buf = self._buf(("gpsend", r), ng * 16)
            ctx.ghost_put_pack(buf if ng else None)
            off, sends[r] = 0, {}
            for p in self.D.peers(r):
                n = self.ghost_recv[r][p]
                sends[r][p] = buf[off * 16:(off + n) * 16]
                off += n
            nsend = sum(n for _, n in self.ghost_seg[r].values())
            rbuf = self._buf(("gprecv", r), nsend * 16)
            rb[r] = (rbuf, nsend)
            recvs[r] = {p: rbuf[o * 16:(o + n) * 16] for p, (o, n) in self.ghost_seg[r].items()}
        self._exchange(sends, recvs)
        for r, ctx in self.m.items():
            rbuf, nsend = rb[r]
            ctx.ghost_put_unpack(rbuf if nsend else None)

    def run(self, nsteps):
        """nsteps velocity-Verlet steps (forces valid on entry and exit)."""
        with self._ctxmgr():
            return self._run(nsteps)

    def _run(self, nsteps):
        from . import pm
        if nsteps <= 0:
            return 0
        flags = {r: ctx.dist_step(self.dt, pm.PM_PHASE_PROLOGUE, read_flag=True)
                 for r, ctx in self.m.items()}
        flag = self._allreduce_max(flags)
        reb = 0
        for s in range(nsteps):
            if flag:
                self._rebuild()
                reb += 1
            elif not self.peer or s == 0:  # peer mode: the sweep refreshed the ghosts
                self._refresh()
            last = s == nsteps - 1
            if self.newton:  # sweep, shares back to the owners, then integrate
                self._newton_forces()
                phase = pm.PM_PHASE_NEWTON_FINAL if last else pm.PM_PHASE_NEWTON_STEP
            else:
                phase = pm.PM_PHASE_FINAL if last else pm.PM_PHASE_STEP
            if self.prof is not None:  # CUDA events around the force/VV kernels
                e0 = self.torch.cuda.Event(enable_timing=True)
                e1 = self.torch.cuda.Event(enable_timing=True)
                e0.record(self.stream)
            if self.sar is not None:  # per-rank sweep times for Stop-At-Rise
                ev = {}
                for r, ctx in self.m.items():
                    a = self.torch.cuda.Event(enable_timing=True)
                    b = self.torch.cuda.Event(enable_timing=True)
                    a.record(self.stream)
                    ctx.dist_step(self.dt, phase, read_flag=False)
                    b.record(self.stream)
                    ev[r] = (a, b)
            else:
                for r, ctx in self.m.items():
                    ctx.dist_step(self.dt, phase, read_flag=False)
            if self.prof is not None:
                e1.record(self.stream)
                self.prof.append((e0, e1))
            if not last:
                flags = {r: ctx.read_flag() for r, ctx in self.m.items()}
            flag = 0 if last else self._allreduce_max(flags)
            if self.sar is not None and not last:
                self.sar.record(self._rank_times({r: a.elapsed_time(b) for r, (a, b) in ev.items()}))
                if self.sar.decide():
                    t0 = time.perf_counter()
                    self.rebalance()
                    self._rebuild()
                    reb += 1
                    self.torch.cuda.synchronize()
                    self.sar.reset(cost=1e3 * (time.perf_counter() - t0))
                    flag = 0  # just rebuilt; the next step refreshes
        return reb

    def _allreduce_min(self, vals):
        v = min(vals.values())
        return v if self.loop else self.tr.allreduce_min_f32(v)

    def dem_start(self):
        """After pm_place and pm_set_dem on every member: DEM state, first
        decomposition, ghosts with velocities and angular velocities."""
        self.dem = True
        with self._ctxmgr():
            for ctx in self.m.values():
                ctx.dist_dem_init()
            self._rebuild()
            self._refresh(pv="pvw")

    def dem_run(self, nsteps, dt):
        """nsteps decomposed DEM steps (pm.h pm_dist_dem_*): contacts +
        leapfrog of the owned grains -> rebuild when any rank asks (contact
        histories migrate with their grains) -> ghost refresh (x, v, omega).
        Returns the number of rebuilds."""
        reb = 0
        with self._ctxmgr():
            for _ in range(nsteps):
                flag = self._allreduce_max({r: ctx.dist_dem_step(dt) for r, ctx in self.m.items()})
                if flag:
                    self._rebuild()
                    reb += 1
                self._refresh(pv="pvw")
        return reb

    def sph_start(self):
        """After pm_place, pm_set_sph and pm_set_rho on every member: start
        the SPH Verlet state, first decomposition, ghosts with velocities."""
        with self._ctxmgr():
            for ctx in self.m.values():
                ctx.dist_sph_init()
            self._rebuild()
            self._refresh(pv=True)

    def sph_run(self, nsteps, cfl=0.2, every=40):
        """nsteps decomposed WCSPH steps (pm.h
        pm_dist_sph_*): local rates -> global min step bound -> update ->
        rebuild when any rank asks -> ghost refresh with velocities.
        Returns (rebuilds, simulated time)."""
        with self._ctxmgr():
            reb, t = 0, 0.0
            for _ in range(nsteps):
                bound = self._allreduce_min({r: ctx.dist_sph_rates() for r, ctx in self.m.items()})
                t += cfl * bound
                flag = self._allreduce_max({r: ctx.dist_sph_update(bound, cfl, every)
                                            for r, ctx in self.m.items()})
                if flag:
                    self._rebuild()
                    reb += 1
                self._refresh(pv=True)
            return reb, t

    def thermo(self):
        """Global KE, U_shift, npairs (sums over ranks)."""
        vals = np.zeros(3)
        for ctx in self.m.values():
            th = ctx.thermo()
            vals += [th["ke"], th["pe_shift"], th["npairs"]]
        if self.newton:  # the energy pass rewrote F without the ghost shares
            with self._ctxmgr():
                self._newton_forces()
        if not self.loop:
            vals = self.tr.allreduce_sum(vals)
        return dict(ke=vals[0], pe_shift=vals[1], npairs=vals[2])


def make_member(system, decomp, rank, device=0, stream=None, rc=2.5, skin=0.3, r_min=0.0,
                sph=None, dem=None):
    """A DistContext for `rank` of `decomp`, with the rank's particles of
    `system` (an inputs.System) placed; `sph` / `dem`: WCSPH / DEM parameters
    (pm_set_sph / pm_set_dem) instead of the LJ ones."""
    from . import pm
    # `stream`: the torch.cuda.Stream the DistSim will run on (never the
    # legacy default stream, whose handle 0 would mean "library-owned stream")
    handle = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
    ctx = pm.DistContext(device=device, stream=handle)
    ctx.set_domain(system.lo, system.hi, system.periodic)
    ctx.set_cutoff(rc, skin)
    if sph is not None:
        ctx.set_sph(sph)
    elif dem is not None:
        ctx.set_dem(dem)
    else:
        ctx.set_lj(1.0, 1.0, 1.0, r_min)
    if decomp.cuts is None:
        ctx.set_decomposition(decomp.grid, decomp.coord(rank))
    else:
        ctx.set_decomposition_cuts(decomp.grid, decomp.coord(rank), decomp.cuts)
    ctx.place(system.pos, system.vel, system.gid, system.kind)
    return ctx


def owner_of(system, decomp):
    """Rank owning each particle (host helper for splitting a generated global
    system; the library applies the same fp32 ownership rule on migration)."""
    lo = system.lo.astype(np.float32)
    L = (system.hi - system.lo).astype(np.float32)
    c = np.zeros((system.n, 3), np.int64)
    for d in range(3):
        p = decomp.grid[d]
        if decomp.cuts is not None:  # slab = number of cuts <= x (fp32 compares)
            cuts = np.asarray(decomp.cuts[d], np.float32)
            c[:, d] = (system.pos[:, d, None] >= cuts[None, :]).sum(axis=1)
            continue
        inv = np.float32(p / float(L[d]))
        u = (system.pos[:, d] - lo[d]).astype(np.float32) * inv
        c[:, d] = np.clip(np.floor(u.astype(np.float32)), 0, p - 1)
    return c[:, 0] + decomp.grid[0] * (c[:, 1] + decomp.grid[1] * c[:, 2])


# ---------------------------------------------------------------- load balancing (NEXT-2)
def weighted_cuts(x, w, p, lo, hi, min_width):
    """Interior cut positions splitting [lo, hi) into p slabs of (nearly) equal
    total weight -- the weighted quantiles k/p of the coordinates x -- then
    moved apart so that every slab is at least min_width wide (PAPER.md:122,
    §3.5: re-balance the work; the per-particle weight is its pair count).
    Returns float32 cuts, increasing."""
    x = np.asarray(x, np.float64)
    w = np.asarray(w, np.float64)
    if p <= 1:
        return np.zeros(0, np.float32)
    if x.size == 0 or w.sum() <= 0:
        cuts = lo + (hi - lo) * np.arange(1, p) / p
    else:
        o = np.argsort(x, kind="stable")
        xs, cw = x[o], np.cumsum(w[o])
        targets = cw[-1] * np.arange(1, p) / p
        k = np.searchsorted(cw, targets)
        cuts = xs[np.minimum(k, xs.size - 1)]
    return _min_width(cuts, p, lo, hi, min_width)


def _min_width(cuts, p, lo, hi, min_width):
    """Move interior cuts apart so that every slab is at least min_width wide
    (forward, then backward pass)."""
    cuts = np.asarray(cuts, np.float64).copy()
    span = hi - lo
    if span < p * min_width * (1 + 1e-6):
        raise ValueError("box too small for p slabs of min_width")
    mw = min_width * (1 + 1e-5)
    for i in range(p - 1):
        cuts[i] = max(cuts[i], (cuts[i - 1] if i else lo) + mw)
    for i in range(p - 2, -1, -1):
        cuts[i] = min(cuts[i], (cuts[i + 1] if i < p - 2 else hi) - mw)
    return cuts.astype(np.float32)


def histogram_cuts(grid, local_pos, local_w, lo, hi, rv, allreduce_sum, bins=4096):
    """Load-balanced tensor-product cuts WITHOUT gathering particles
    (§3.5): every rank bins its owned particles' coordinates,
    weighted by their pair work, into `bins` slabs per decomposed axis; the
    histograms are summed over ranks (allreduce_sum) and every rank cuts the
    same global histogram at the weighted quantiles k/p (upper edge of the
    crossing bin), then enforces slabs >= 2 r_v.  Identical cuts on every
    rank."""
    local_pos = np.asarray(local_pos, np.float64).reshape(-1, 3)
    local_w = np.asarray(local_w, np.float64).reshape(-1)
    hs = []
    for d in range(3):
        h, _ = np.histogram(local_pos[:, d], bins=bins, range=(float(lo[d]), float(hi[d])),
                            weights=local_w)
        hs.append(h)
    H = np.asarray(allreduce_sum(np.concatenate(hs)), np.float64).reshape(3, bins)
    cuts = []
    for d in range(3):
        p = grid[d]
        if p <= 1:
            cuts.append(np.zeros(0, np.float32))
            continue
        edges = np.linspace(float(lo[d]), float(hi[d]), bins + 1)
        cw = np.cumsum(H[d])
        if cw[-1] <= 0:
            c = float(lo[d]) + (float(hi[d]) - float(lo[d])) * np.arange(1, p) / p
        else:
            k = np.searchsorted(cw, cw[-1] * np.arange(1, p) / p)
            c = edges[np.minimum(k + 1, bins)]
        cuts.append(_min_width(c, p, float(lo[d]), float(hi[d]), 2.0 * float(rv) * (1 + 1e-5)))
    return tuple(cuts)


def balanced_decomp(grid, pos, weights, lo, hi, rv):
    """Tensor-product load-balanced cuts: per axis, weighted quantiles of all
    particles' coordinates (identical on every rank given the same global
    data, e.g. all-reduced histograms)."""
    cuts = tuple(weighted_cuts(pos[:, d], weights, grid[d], float(lo[d]), float(hi[d]),
                               2.0 * rv * (1 + 1e-5)) for d in range(3))
    return Decomp(tuple(grid), cuts)


def imbalance(work):
    """max / mean of the per-rank work (1.0 = perfectly balanced)."""
    work = np.asarray(list(work), np.float64)
    return float(work.max() / work.mean()) if work.size and work.mean() > 0 else 1.0


class SAR:
    """Stop-At-Rise re-balancing trigger (PAPER.md:122 '[56]'):
    per step record the degradation delta = max - mean of the per-rank step
    times; W(n) = (C + sum delta) / n with C the cost of a re-balance;
    re-balance at the first rise W(n) > W(n-1) (W(0) = +inf); at most one
    True per reset (the caller re-balances and calls reset)."""

    def __init__(self, cost):
        self.C = float(cost)
        self.reset()

    def reset(self, cost=None):
        if cost is not None:
            self.C = float(cost)
        self.n, self.sum, self.W = 0, 0.0, float("inf")
        self.fired = False

    def record(self, per_rank_times):
        t = np.asarray(per_rank_times, np.float64)
        self.sum += float(t.max() - t.mean())
        self.n += 1

    def decide(self):
        if self.fired or self.n == 0:
            return False
        W = (self.C + self.sum) / self.n
        rise = W > self.W
        self.W = W
        self.fired = rise
        return rise


# ---------------------------------------------------------------- bench (N>1)
def _grid_for(n):
    return {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}.get(n) or (n, 1, 1)


def bench_main(args):
    """bench.py --gpus N under torchrun.  Default: the native group path
    (pm_create_dist / pm_map / pm_ghost_get / pm_dist_run behind the C-ABI,
    library-owned NCCL communicator); PM_DIST_NATIVE=0: the Python DistSim
    orchestration over torch.distributed (bench_distsim)."""
    if os.environ.get("PM_DIST_NATIVE", "1") != "0":
        return bench_native(args)
    return bench_distsim(args)


def bench_native(args):
    """BJ configs[2] weak scaling through the C-ABI group API: one 128^3
    lattice block (2,097,152 particles) per GPU; the unique id travels over a
    gloo process group (bootstrap only: every data-path byte and the per-step
    flag all-reduce go through the library's NCCL communicator).
    PM_CFG3_BLOCK=m: m^3 particles per rank."""
    import torch
    import torch.distributed as tdist
    from . import build as pmbuild, inputs, pm
    pmbuild.build()
    ws = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    m = int(os.environ.get("PM_CFG3_BLOCK", "128"))
    dev = local % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    tdist.init_process_group("gloo")
    grid = _grid_for(ws)
    D = Decomp(grid)
    s = inputs.cfg3_block(*D.coord(rank), grid=grid, m=m)
    stream = torch.cuda.Stream()

    def max_f(x):
        t = torch.tensor([float(x)], dtype=torch.float64)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        return float(t.item())

    def sum_i(x):
        t = torch.tensor([int(x)], dtype=torch.int64)
        tdist.all_reduce(t)
        return int(t.item())

    def member(place=True):
        # a fresh unique id per communicator (an id bootstraps one init only)
        uid = [pm.nccl_unique_id() if rank == 0 else None]
        tdist.broadcast_object_list(uid, src=0)
        c = pm.create_dist(rank, ws, uid[0], grid, device=dev, stream=stream.cuda_stream)
        c.set_domain(s.lo, s.hi, s.periodic)
        c.set_cutoff(2.5, 0.3)
        c.set_lj(1.0, 1.0, 1.0, 0.0)
        if place:
            c.place(s.pos, s.vel, s.gid)
        return c

    # ---- device-resident run (value)
    c = member()
    c.map()
    c.ghost_get()
    c.dist_run(0.005, args.warmup)
    torch.cuda.synchronize()
    tdist.barrier()
    clocks = None
    if rank == 0:
        from bench import ClockSampler  # noqa: E402
        clocks = ClockSampler(dev)
        clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    r = c.dist_run(0.005, args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    tdist.barrier()
    clk = clocks.stop() if clocks else None
    ms = max_f(e0.elapsed_time(e1))
    cnt = c.count()
    n = sum_i(cnt["n_owned"])
    # dominant kernel (force sweep + fused VV): events around every step's
    # sweep inside pm_dist_run (pm_set_profiling), max over ranks
    c.set_profiling(True)
    c.dist_run(0.005, min(args.steps, 50))
    prof = c.get_profile()
    c.set_profiling(False)
    sweep_ms = max_f(prof["force_ms"] / max(prof["force_launches"], 1))
    nbar = cnt["nnz"] / max(cnt["n_owned"], 1)
    alg = cnt["n_owned"] * (4.0 * nbar + 64.0)
    c.close()
    # ---- end to end: pinned host state in, K steps, owned state out
    pos_h = torch.from_numpy(s.pos).pin_memory()
    vel_h = torch.from_numpy(s.vel).pin_memory()
    gid_h = torch.from_numpy(s.gid).pin_memory()
    c = member(place=False)
    torch.cuda.synchronize()
    tdist.barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    c.place(pos_h, vel_h, gid_h)
    c.map()
    c.ghost_get()
    c.dist_run(0.005, args.steps)
    out = c.owned_state()
    t1.record(stream)
    torch.cuda.synchronize()
    tdist.barrier()
    e2e_ms = max_f(t0.elapsed_time(t1))
    c.close()
    if rank == 0:
        from bench import METRIC, UNIT, hbm_peak  # noqa: E402
        h2d = s.n * (16 + 16 + 8)
        d2h = int(out["pos"].nbytes + out["vel"].nbytes)
        peak, peak_src = hbm_peak()
        ach = alg / (sweep_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": ach / peak, "traffic": None,
                "kernel": "k_lj_step (force sweep + fused VV), rank 0 sub-domain",
                "kernel_ms": sweep_ms, "kernel_share_of_step": sweep_ms / (ms / args.steps),
                "alg_bytes_per_launch": alg, "alg_bytes_formula": "N_owned*(4*nbar + 64)",
                "peak_source": peak_src}
        line = {"metric": METRIC, "value": n * args.steps / (ms * 1e-3), "unit": UNIT,
                "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": f"cfg3 (BJ configs[2]): LJ fluid, {m**3:,} particles per "
                                       f"GPU (SC {m}^3 block, rho=0.8), cuboid decomposition "
                                       f"{grid}, ghost width r_cut+skin, NVE",
                           "n_particles": n, "parallelism": f"spatial {grid} (NCCL, native "
                                                            "pm_dist_run)",
                           "rebuilds": r["rebuilds"], "l2": "inputs larger than L2 (Verlet lists)"},
                "roofline": roof, "cpu_baseline": None,
                "e2e": {"value": n * args.steps / (e2e_ms * 1e-3), "unit": UNIT,
                        "h2d_bytes_per_step": h2d * ws / args.steps,
                        "d2h_bytes_per_step": d2h * ws / args.steps},
                # per step: refresh pack + unpack, sweep, pending flip (+ NCCL
                # send/recv) = 4; per rebuild: 2 x (plan 4 + pack + unpack) +
                # compact + flip + build 11 + remap = 26
                "gpu_launches": 4 * args.steps + 26 * r["rebuilds"] + 3, "clocks": clk}
        print(json.dumps(line), flush=True)
    tdist.destroy_process_group()
    return 0


def bench_distsim(args):
    """bench.py --gpus N under torchrun: BJ configs[2] weak scaling, one
    128^3 lattice block (2,097,152 particles) per GPU, NCCL transport.
    PM_DIST_BACKEND=gloo (tests only): ranks may share a GPU, messages are
    staged through host memory.  PM_CFG3_BLOCK=m: m^3 particles per rank."""
    import torch
    import torch.distributed as tdist
    from . import build as pmbuild, inputs
    pmbuild.build()
    ws = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    backend = os.environ.get("PM_DIST_BACKEND", "nccl")
    m = int(os.environ.get("PM_CFG3_BLOCK", "128"))
    dev = local % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    if backend == "nccl":
        tdist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        tr = TorchTransport(device=torch.device("cuda", dev))
        red_dev = "cuda"
    else:
        tdist.init_process_group("gloo")
        tr = TorchTransport(device=None, stage_host=True)
        red_dev = "cpu"
    D = Decomp(_grid_for(ws))
    s = inputs.cfg3_block(*D.coord(rank), grid=D.grid, m=m)
    stream = torch.cuda.Stream()

    def max_ms(ms):
        t = torch.tensor([ms], dtype=torch.float64, device=red_dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident run (value)
    ctx = make_member(s, D, rank, device=dev, stream=stream)
    sim = DistSim(D, {rank: ctx}, tr, stream=stream)
    sim.start()
    sim.run(args.warmup)
    torch.cuda.synchronize()
    tdist.barrier()
    clocks = None
    if rank == 0:
        from bench import ClockSampler  # noqa: E402
        clocks = ClockSampler(dev)
        clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    reb = sim.run(args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    tdist.barrier()
    clk = clocks.stop() if clocks else None
    ms = max_ms(e0.elapsed_time(e1))
    cnt = ctx.count()
    n_tot = torch.tensor([cnt["n_owned"]], dtype=torch.int64, device=red_dev)
    tdist.all_reduce(n_tot)
    n = int(n_tot.item())
    # dominant kernel (the fused force sweep + VV), a second pass timed with
    # events around each step's sweep on this rank's stream; max over ranks
    sim.prof = []
    sim.run(min(args.steps, 50))
    torch.cuda.synchronize()
    sweep_ms = sum(a.elapsed_time(b) for a, b in sim.prof) / len(sim.prof)
    sim.prof = None
    sweep_ms = max_ms(sweep_ms)
    nbar = cnt["nnz"] / max(cnt["n_owned"], 1)
    alg = cnt["n_owned"] * (4.0 * nbar + 64.0)
    ctx.close()
    # ---- end to end: pinned host state in, K steps, owned state out
    pos_h = torch.from_numpy(s.pos).pin_memory()
    vel_h = torch.from_numpy(s.vel).pin_memory()
    gid_h = torch.from_numpy(s.gid).pin_memory()
    ctx = make_member(s, D, rank, device=dev, stream=stream)
    sim = DistSim(D, {rank: ctx}, tr, stream=stream)
    torch.cuda.synchronize()
    tdist.barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    ctx.place(pos_h, vel_h, gid_h)
    with torch.cuda.stream(stream):
        sim.start()
        sim.run(args.steps)
    out = ctx.owned_state()
    t1.record(stream)
    torch.cuda.synchronize()
    tdist.barrier()
    e2e_ms = max_ms(t0.elapsed_time(t1))
    ctx.close()
    if rank == 0:
        from bench import METRIC, UNIT  # noqa: E402
        h2d = s.n * (16 + 16 + 8)
        d2h = int(out["pos"].nbytes + out["vel"].nbytes)
        from bench import hbm_peak  # noqa: E402
        peak, peak_src = hbm_peak()
        ach = alg / (sweep_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": ach / peak, "traffic": None,
                "kernel": "k_lj_step (force sweep + fused VV), rank 0 sub-domain",
                "kernel_ms": sweep_ms, "kernel_share_of_step": sweep_ms / (ms / args.steps),
                "alg_bytes_per_launch": alg, "alg_bytes_formula": "N_owned*(4*nbar + 64)",
                "peak_source": peak_src}
        line = {"metric": METRIC, "value": n * args.steps / (ms * 1e-3), "unit": UNIT,
                "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": f"cfg3 (BJ configs[2]): LJ fluid, {m**3:,} particles per "
                                       f"GPU (SC {m}^3 block, rho=0.8), cuboid decomposition "
                                       f"{D.grid}, ghost width r_cut+skin, NVE",
                           "n_particles": n, "parallelism": f"spatial {D.grid} ({backend})",
                           "rebuilds": reb, "l2": "inputs larger than L2 (Verlet lists)"},
                "roofline": roof, "cpu_baseline": None,
                "e2e": {"value": n * args.steps / (e2e_ms * 1e-3), "unit": UNIT,
                        "h2d_bytes_per_step": h2d * ws / args.steps,
                        "d2h_bytes_per_step": d2h * ws / args.steps},
                # per step: refresh pack + unpack, sweep, flag clear (+1 apply)
                # = 5; per rebuild: 2 x (plan 4 + pack + unpack) + compact +
                # flip + build 11 + remap = 26; prologue and start 3
                "gpu_launches": 5 * args.steps + 26 * reb + 3, "clocks": clk}
        print(json.dumps(line), flush=True)
    tdist.destroy_process_group()
    return 0
