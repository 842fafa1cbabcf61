"""Two processes, one GPU, CUDA-IPC fused ghost refresh (DistSim(peer=True)
over a gloo process group): each rank owns one cfg3 block of a (2,1,1)
decomposition; the force sweep's epilogue stores every new position of a
sent particle straight into the OTHER process's ghost slots through CUDA IPC
mappings.  After 40 steps (with rebuilds) rank 0 compares the union of the
owned states with one context on the global system and prints
"peer-ipc OK ...".  Usage: torchrun --nproc-per-node 2 tools/dist_peer_check.py [m]"""
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
torch.cuda.set_device(0)
tdist.init_process_group("gloo")
D = dist.Decomp((ws, 1, 1))
s = inputs.cfg3_block(*D.coord(rank), grid=D.grid, m=m)
stream = torch.cuda.Stream()
ctx = dist.make_member(s, D, rank, stream=stream)
sim = dist.DistSim(D, {rank: ctx}, dist.TorchTransport(device=None, stage_host=True),
                   stream=stream, peer=True)
sim.start()
reb = sim.run(40)
st = ctx.owned_state()
parts = [None] * ws
tdist.all_gather_object(parts, {k: st[k] for k in ("gid", "pos", "vel")})
if rank == 0:
    g = inputs.cfg3_global(D.grid, m=m)
    ref = pm.Context()
    ref.set_domain(g.lo, g.hi, g.periodic)
    ref.set_cutoff(2.5, 0.3)
    ref.set_lj(1.0, 1.0, 1.0, 0.0)
    ref.place(g.pos, g.vel, g.gid)
    ref.step_vv(0.005, 40)
    rst = pm.sorted_by_gid(ref.get_state())
    got = pm.sorted_by_gid({k: np.concatenate([p[k] for p in parts]) for k in parts[0]})
    assert np.array_equal(got["gid"], np.sort(g.gid))
    L = g.hi.astype(np.float64)
    d = got["pos"][:, :3].astype(np.float64) - rst["pos"][:, :3]
    d -= L * np.round(d / L)
    dv = np.max(np.abs(got["vel"][:, :3] - rst["vel"][:, :3]))
    assert np.max(np.abs(d)) < 1e-3 and dv < 1e-2, (np.max(np.abs(d)), dv)
    print(f"peer-ipc OK ws={ws}: {reb} rebuilds, max |dx| {np.max(np.abs(d)):.2e}, "
          f"max |dv| {dv:.2e}", flush=True)
tdist.barrier()
ctx.ipc_close_all()
ctx.close()
tdist.destroy_process_group()
