"""One cfg-3 IK solve (for ncu): 300 goals x 30 seeds x 100 iterations, shared K = 20 scene."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_17274_b200 import native, workload
wl = workload.franka_ik(0, list(range(300)), S=30, iters=100)
ctx = native.Context(0)
ctx.set_robot(wl.robot); ctx.set_world(wl.worlds); ctx.set_cost_params(wl.cost)
ctx.solve(wl.solver, torch.tensor(wl.seeds, device="cuda"), torch.tensor(wl.goal, device="cuda"),
          env=torch.tensor(wl.env, device="cuda"))
torch.cuda.synchronize()
print("done")
