import sys, dataclasses
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2310_17274_b200 import native, motion_gen, workload
P = 64
wl = workload.franka_to(0, list(range(P)), S=12, H=32, iters=100)
T = lambda a, dt=torch.float32: torch.tensor(np.ascontiguousarray(a), dtype=dt, device="cuda")
for name, kw in [("base", {}), ("bw4", {"beta_world": 4 * wl.cost.beta_world}), ("a0/4", {"a0": wl.cost.a0 / 4}),
                 ("eta.05", {"eta": 0.05}), ("nospeed", {"flags": wl.cost.flags & ~2})]:
    cost = dataclasses.replace(wl.cost, **kw)
    ctx = native.Context(0); ctx.set_robot(wl.robot); ctx.set_world(wl.worlds); ctx.set_cost_params(cost)
    mg = motion_gen.MotionGen(ctx, wl.robot, cost)
    out = mg.plan(T(wl.start), T(wl.goal), T(wl.env, torch.int32), T(mg.ik_seed_batch(wl.robot, range(P), 32)))
    pe = out["pos_err"].cpu().numpy(); re = out["rot_err"].cpu().numpy()
    H = 32
    v = ctx.mask_samples(out["traj"].view(P * H, 7), env=T(wl.env, torch.int32), env_div=H).view(P, H).cpu().numpy()
    allv = v.all(1)
    print(name, "success", int(out["success"].sum()), "pose_ok", int(((pe < 5e-3) & (re < 0.05)).sum()), "valid", int(allv.sum()),
          "ik_count>0", int((out["ik_count"].cpu().numpy() > 0).sum()), flush=True)
    ctx.close()
