"""Small solves for compute-sanitizer (memcheck / racecheck / synccheck): sequential and cluster
TO and IK with particles, both world builds."""
import os, sys, dataclasses
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_17274_b200 import native, workload, inputs
for big in (False, True):
    wl = workload.franka_to(0, [0], S=2, H=16, iters=3, n_boxes=70 if big else 20)
    ctx = native.Context(0)
    ctx.set_robot(wl.robot); ctx.set_world(wl.worlds); ctx.set_cost_params(wl.cost)
    for c in (0, 1):
        sp = dataclasses.replace(wl.solver, particle_iters=1, n_particles=8, cluster=c)
        ctx.solve(sp, torch.tensor(wl.seeds, device="cuda"), torch.tensor(wl.goal, device="cuda"),
                  start=torch.tensor(wl.start, device="cuda"), env=torch.tensor(wl.env, device="cuda"))
    torch.cuda.synchronize()
    ctx.close()
wl = workload.franka_ik(0, [0, 1], S=30, iters=3)
ctx = native.Context(0)
ctx.set_robot(wl.robot); ctx.set_world(wl.worlds); ctx.set_cost_params(wl.cost)
for c in (0, 1):
    sp = dataclasses.replace(wl.solver, particle_iters=1, n_particles=8, cluster=c)
    ctx.solve(sp, torch.tensor(wl.seeds, device="cuda"), torch.tensor(wl.goal, device="cuda"),
              env=torch.tensor(wl.env, device="cuda"))
torch.cuda.synchronize()
print("done")
