"""Multi-process check of the native group path (pm_create_dist: one member
per process, library-owned NCCL communicator) under torchrun: every rank
places its cfg3 block, pm_map / pm_ghost_get / pm_dist_run, then rank 0
compares the union of the owned states with one context on the global system.
Usage: torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/dist_native_check.py [m]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as tdist  # noqa: E402
from paper_1804_07598_b200 import build, dist, inputs, pm  # noqa: E402

build.build()
m = int(sys.argv[1]) if len(sys.argv) > 1 else 24
ws, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
dev = int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count()
torch.cuda.set_device(dev)
tdist.init_process_group("gloo")
grid = dist._grid_for(ws)
uid = [pm.nccl_unique_id() if rank == 0 else None]
tdist.broadcast_object_list(uid, src=0)
c = pm.create_dist(rank, ws, uid[0], grid, device=dev)
D = dist.Decomp(grid)
s = inputs.cfg3_block(*D.coord(rank), grid=grid, m=m)
c.set_domain(s.lo, s.hi, s.periodic)
c.set_cutoff(2.5, 0.3)
c.set_lj(1.0, 1.0, 1.0, 0.0)
c.place(s.pos, s.vel, s.gid)
c.map()
c.ghost_get()
r = c.dist_run(0.005, 30)
th = c.dist_thermo()
st = c.owned_state()
parts = [None] * ws
tdist.all_gather_object(parts, {k: st[k] for k in ("gid", "pos", "vel")})
if rank == 0:
    g = inputs.cfg3_global(grid, m=m)
    ref = pm.Context(device=dev)
    ref.set_domain(g.lo, g.hi, g.periodic)
    ref.set_cutoff(2.5, 0.3)
    ref.set_lj(1.0, 1.0, 1.0, 0.0)
    ref.place(g.pos, g.vel, g.gid)
    rr = ref.step_vv(0.005, 30)
    rst = pm.sorted_by_gid(ref.get_state())
    got = pm.sorted_by_gid({k: np.concatenate([p[k] for p in parts]) for k in parts[0]})
    assert np.array_equal(got["gid"], np.sort(g.gid))
    L = g.hi.astype(np.float64)
    d = got["pos"][:, :3].astype(np.float64) - rst["pos"][:, :3]
    d -= L * np.round(d / L)
    thr = ref.thermo()
    print(f"native dist check ws={ws} grid={grid}: steps {r['steps']} rebuilds {r['rebuilds']} "
          f"(single {rr['rebuilds']}), max |dx| {np.max(np.abs(d)):.2e}, npairs "
          f"{th['npairs']} vs {thr['npairs']}, ke {th['ke']:.6f} vs {thr['ke']:.6f}")
    assert np.max(np.abs(d)) < 1e-3 and th["npairs"] == thr["npairs"]
c.close()
tdist.destroy_process_group()
