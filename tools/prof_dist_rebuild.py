"""cProfile of DistSim rebuilds (loopback, cfg3 (2,1,1)): where the host time of
a decomposed rebuild goes.  Usage: python tools/prof_dist_rebuild.py"""
import cProfile, pstats, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1804_07598_b200 import dist, inputs, pm
grid=(2,1,1)
s = inputs.cfg3_global(grid=grid, m=128)
D = dist.Decomp(grid)
owner = dist.owner_of(s, D)
stream = torch.cuda.Stream()
members = {q: dist.make_member(s.subset(np.where(owner == q)[0]), D, q, stream=stream) for q in range(D.size)}
sim = dist.DistSim(D, members, dist.LoopbackTransport(members), stream=stream)
sim.start(); sim.run(20); torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(10):
    sim.rebuild()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
