"""BJ configs[4] (clustered LJ, reading R22 capped force) on ONE GPU:

 * frozen mode (SURVEY §8(d) cfg5 secondary): `reps` repeats of cell list +
   Verlet build + capped-LJ force pass on the fixed clustered configuration,
   CUDA events around each phase; PU/s = N / t_pass; pairs/s; the force
   sweep's algorithmic HBM fraction (N (4 nbar + 16 + 16) bytes: list, count,
   position read, force write);
 * the 2x2x2 split (loopback, 8 sub-domains on this GPU): per sub-domain
   owned N, list entries and sweep time with equal cuts and with the
   load-balanced cuts from all-reduced pair-work histograms (NEXT-2).

Full cfg5 is 64 clusters x 131,072 (8.4M particles, ~3.5e10 list entries =
142 GB: the 8-GPU case); this tool keeps the cluster shape (131,072 per
cluster, sigma_c = 4, rho = 0.5 overall -- the same local density, rows up
to ~12k) with `nc` clusters (default 8: 1,048,576 particles, one GPU's share).
Usage: python tools/cfg5_bench.py [nc] [reps] > out.json"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1804_07598_b200 import build, dist, inputs, pm  # noqa: E402

build.build()
nc = int(sys.argv[1]) if len(sys.argv) > 1 else 8
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
s = inputs.cfg5(n_clusters=nc)
stream = torch.cuda.Stream()
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
c = pm.Context(stream=stream.cuda_stream)
c.set_domain(s.lo, s.hi, s.periodic)
c.set_cutoff(2.5, 0.3)
c.set_lj(1.0, 1.0, 1.0, 0.8)
c.place(s.pos, s.vel, s.gid)
c.build_verlet()  # sizes the SELL layout from the exact counts (overflow + retry)
c.compute_lj()
tb, tf = [], []
for _ in range(reps):
    e0, e1, e2 = ev(), ev(), ev()
    torch.cuda.synchronize()
    e0.record(stream)
    c.build_verlet()
    e1.record(stream)
    c.compute_lj()
    e2.record(stream)
    torch.cuda.synchronize()
    tb.append(e0.elapsed_time(e1))
    tf.append(e0.elapsed_time(e2) - e0.elapsed_time(e1))
cnt = c.count()
th = c.thermo(recompute=True)
rp, _ = c.get_verlet(cols=False)
gid = c.get_state()["gid"]
w = np.zeros(s.n)
w[gid] = np.diff(rp)
c.close()
nnz = cnt["nnz"]
build_ms, force_ms = float(np.median(tb)), float(np.median(tf))
pass_ms = build_ms + force_ms
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists("MEASURED_PEAKS.json") else 6548.8
alg = s.n * (4.0 * nnz / s.n + 16 + 16)
out = {"workload": f"cfg5-class clustered LJ: {nc} Gaussian clusters x 131,072 (sigma_c 4, "
                   f"rho 0.5 overall; BJ configs[4] local density), capped LJ r_min 0.8",
       "n_particles": s.n, "frozen": {
           "repeats": reps, "build_ms": build_ms, "force_ms": force_ms, "pass_ms": pass_ms,
           "value": s.n / (pass_ms * 1e-3), "unit": "particle-updates/s (bin + list + force)",
           "list_entries": nnz, "mean_row": nnz / s.n, "max_row": int(np.max(np.diff(rp))),
           "pairs_in_rc": int(th["npairs"]), "pair_interactions_per_s": th["npairs"] / (pass_ms * 1e-3),
           "force_sweep_roofline": {"bound": "hbm", "achieved": alg / (force_ms * 1e-3) / 1e9,
                                    "peak": peak, "unit": "GB/s",
                                    "frac": alg / (force_ms * 1e-3) / 1e9 / peak,
                                    "alg_bytes": alg,
                                    "formula": "N (4 nbar + 16 + 16): list, counts, x read, F write"}}}
# ---- 2x2x2 split in loopback: equal cuts vs load-balanced cuts
grid = (2, 2, 2)
split = {}
for name in ("equal", "balanced"):
    if name == "equal":
        D = dist.Decomp(grid)
    else:
        cuts = dist.histogram_cuts(grid, s.pos[:, :3], w + 1.0, s.lo, s.hi, 2.8,
                                   lambda h: h)
        D = dist.Decomp(grid, cuts)
    owner = dist.owner_of(s, D)
    members = {r: dist.make_member(s.subset(np.where(owner == r)[0]), D, r, stream=stream,
                                   r_min=0.8) for r in range(D.size)}
    sim = dist.DistSim(D, members, dist.LoopbackTransport(members), stream=stream)
    sim.start()
    times = []
    for r, ctx in members.items():  # each sub-domain's force sweep alone
        a, b = ev(), ev()
        torch.cuda.synchronize()
        a.record(stream)
        ctx.dist_step(0.005, pm.PM_PHASE_FORCES)
        b.record(stream)
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
    n_own = [ctx.count()["n_owned"] for ctx in members.values()]
    nz = [ctx.count()["nnz"] for ctx in members.values()]
    split[name] = {"cuts": None if D.cuts is None else [list(map(float, x)) for x in D.cuts],
                   "n_owned": n_own, "list_entries": nz, "sweep_ms": times,
                   "imbalance_entries": dist.imbalance(nz), "imbalance_sweep_ms": dist.imbalance(times)}
    for ctx in members.values():
        ctx.close()
out["split_2x2x2"] = split
print(json.dumps(out))
