"""Stage-by-stage diagnostics of the motion-generation pipeline (f2) on a few problems."""
import sys
import numpy as np
import torch
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2310_17274_b200 import native, motion_gen, workload  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 6
dev = torch.device("cuda:0")
wl = workload.franka_to(0, list(range(P)), S=12, H=32, iters=100)
ctx = native.Context(0)
import dataclasses, os
cost = dataclasses.replace(wl.cost, a1=wl.cost.a1 * float(os.environ.get("A1X", "1")),
                           a0=wl.cost.a0 * float(os.environ.get("A0X", "1")))
ctx.set_robot(wl.robot); ctx.set_world(wl.worlds); ctx.set_cost_params(cost)
cfg = motion_gen.MotionGenConfig(**({"rot_thr": float(os.environ["ROT"])} if "ROT" in os.environ else {}))
mg = motion_gen.MotionGen(ctx, wl.robot, cost, cfg)
T = lambda a, dt=torch.float32: torch.tensor(np.ascontiguousarray(a), dtype=dt, device=dev)
out = mg.plan(T(wl.start), T(wl.goal), T(wl.env, torch.int32), T(mg.ik_seed_batch(wl.robot, range(P), 32)))
torch.cuda.synchronize()
np.set_printoptions(precision=4, suppress=True, linewidth=160)
print("success", out["success"].cpu().numpy(), "A1X", os.environ.get("A1X"), "ROT", os.environ.get("ROT"))
print("ik_count", out["ik_count"].cpu().numpy())
print("to1 score", out["to1_score"].cpu().numpy())
print("best1", out["best1"].cpu().numpy().ravel(), "dt_opt", out["dt_opt"].cpu().numpy())
print("final pos_err", out["pos_err"].cpu().numpy(), "rot_err", out["rot_err"].cpu().numpy())
print("final dt", out["dt"].cpu().numpy(), "max_jerk", out["max_jerk"].cpu().numpy())
H, D = 32, 7
tr2 = out["traj"]
v2 = ctx.mask_samples(tr2.view(P * H, D), env=T(wl.env, torch.int32), env_div=H).view(P, H).cpu().numpy()
print("final state validity per problem", v2.sum(1))
tr1 = out["to1_traj"]
pe1, re1 = ctx.goal_error(tr1.view(-1)[(H - 1) * D:], T(wl.goal), B=P * 12, stride=H * D, goal_div=12)
print("to1 pos_err", pe1.view(P, 12).cpu().numpy())
print("to1 rot_err", re1.view(P, 12).cpu().numpy())
v1 = ctx.mask_samples(tr1.view(P * 12 * H, D), env=T(wl.env, torch.int32), env_div=12 * H).view(P, 12, H).cpu().numpy()
print("to1 valid states", v1.sum(2))
envt = T(wl.env, torch.int32)
# mask_samples evaluates 32 rows per CTA against ONE environment (rows of a group share env[row //
# env_div]): one call per problem here, since every problem has its own scene
print("start valid", [int(ctx.mask_samples(T(wl.start[p:p + 1]), env=envt[p:p + 1]).item()) for p in range(P)])
b1 = out["best1"].cpu().numpy().ravel()
for p in range(P):
    print("p", p, "to1 best state validity", v1[p, b1[p]].astype(int))
ik = out["ik_q"]
pe, re = ctx.goal_error(ik, T(wl.goal), B=P * 32, goal_div=32)
print("ik pos_err min/med", pe.view(P, 32).min(1).values.cpu().numpy(), pe.view(P, 32).median(1).values.cpu().numpy())
print("ik rot_err min/med", re.view(P, 32).min(1).values.cpu().numpy(), re.view(P, 32).median(1).values.cpu().numpy())
vi = ctx.mask_samples(ik.view(P * 32, 7), env=envt, env_div=32).view(P, 32).cpu().numpy()
print("ik valid", vi.sum(1))
