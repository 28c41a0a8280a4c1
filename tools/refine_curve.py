import sys, dataclasses
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2310_17274_b200 import native, motion_gen, workload, inputs
P = 8
wl = workload.franka_to(0, list(range(P)), S=12, H=32, iters=100)
T = lambda a, dt=torch.float32: torch.tensor(np.ascontiguousarray(a), dtype=dt, device="cuda")
ctx = native.Context(0); ctx.set_robot(wl.robot); ctx.set_world(wl.worlds); ctx.set_cost_params(wl.cost)
mg = motion_gen.MotionGen(ctx, wl.robot, wl.cost)
st, gl, env = T(wl.start), T(wl.goal), T(wl.env, torch.int32)
out = mg.plan(st, gl, env, T(mg.ik_seed_batch(wl.robot, range(P), 32)))
H, D = 32, 7
seed2 = motion_gen.N.gather_rows(out["to1_traj"].view(P, 12, H * D), out["best1"]).view(P, 1, H, D) if hasattr(motion_gen, "N") else None
from paper_2310_17274_b200 import native as N
seed2 = N.gather_rows(out["to1_traj"].view(P, 12, H * D), out["best1"]).view(P, 1, H, D)
ctx.set_cost_params(mg.cost_to2)
rows = []
for k in range(0, 301, 25):
    o = ctx.solve(dataclasses.replace(mg.sp_refine, iters=k, check_every=0), seed2, gl, start=st, env=env, dt=out["dt_opt"])
    rows.append(o["best_cost"].cpu().numpy())
np.set_printoptions(precision=3, suppress=True, linewidth=200)
print(np.array(rows))
