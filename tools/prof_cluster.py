"""One latency-mode solve for ncu: 8 problems x 32 seeds x 32 timesteps x 100 iterations (cluster
of 4 CTAs per seed), K = 20."""
import os, sys, dataclasses
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_17274_b200 import native, workload
wl = workload.franka_to(0, list(range(8)), S=32, H=32, iters=100)
ctx = native.Context(0)
ctx.set_robot(wl.robot); ctx.set_world(wl.worlds); ctx.set_cost_params(wl.cost)
ctx.solve(dataclasses.replace(wl.solver, cluster=1), torch.tensor(wl.seeds, device="cuda"),
          torch.tensor(wl.goal, device="cuda"), start=torch.tensor(wl.start, device="cuda"),
          env=torch.tensor(wl.env, device="cuda"))
torch.cuda.synchronize()
print("done")
