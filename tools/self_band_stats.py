"""Fraction of self-collision pairs (S) within a band of d^2 - R^2 along seeds and solved
trajectories of the bench workload (analysis tool: how many pairs a coarser screen would flag)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2310_17274_b200 import native, workload

wl = workload.franka_to(0, list(range(8)), S=32, H=32, iters=100)
ctx = native.Context(0)
ctx.set_robot(wl.robot); ctx.set_world(wl.worlds); ctx.set_cost_params(wl.cost)
out = ctx.solve(wl.solver, torch.tensor(wl.seeds, device="cuda"), torch.tensor(wl.goal, device="cuda"),
                start=torch.tensor(wl.start, device="cuda"), env=torch.tensor(wl.env, device="cuda"),
                seed_outputs=True)
rb = wl.robot
pairs = np.asarray(rb.pairs)
r = np.asarray(rb.spheres)[:, 3]
ok = (r[pairs[:, 0]] > 0) & (r[pairs[:, 1]] > 0)
pairs = pairs[ok]
R = r[pairs[:, 0]] + r[pairs[:, 1]]
for name, q in (("seeds", wl.seeds.reshape(-1, 7)), ("solved", out["seed_best_traj"].cpu().numpy().reshape(-1, 7))):
    sph, _ = ctx.fk(torch.tensor(q, device="cuda", dtype=torch.float32))
    w = sph[:, :, :3].cpu().numpy().astype(np.float64)
    d2 = ((w[:, pairs[:, 0]] - w[:, pairs[:, 1]]) ** 2).sum(-1)
    m = d2 - R[None] ** 2
    print(name, "configs", len(q), " ".join(f"<{b:g}: {np.mean(m < b):.4f}" for b in (0, 2e-5, 1e-3, 2e-3, 4e-3, 8e-3)))
ctx.close()
