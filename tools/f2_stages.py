import sys, dataclasses, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2310_17274_b200 import native, motion_gen, workload, inputs
for P in (1, 64):
    wl = workload.franka_to(0, list(range(P)), S=12, H=32, iters=100)
    T = lambda a, dt=torch.float32: torch.tensor(np.ascontiguousarray(a), dtype=dt, device="cuda")
    ctx = native.Context(0); ctx.set_robot(wl.robot); ctx.set_world(wl.worlds); ctx.set_cost_params(wl.cost)
    mg = motion_gen.MotionGen(ctx, wl.robot, wl.cost)
    st, gl, env = T(wl.start), T(wl.goal), T(wl.env, torch.int32)
    seeds_ik = T(mg.ik_seed_batch(wl.robot, range(P), 32))
    mg.plan(st, gl, env, seeds_ik); torch.cuda.synchronize()
    # stage timings by wrapping ctx.solve
    orig = ctx.solve
    log = []
    def timed(*a, **k):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); r = orig(*a, **k); e1.record(); log.append((a[1].shape, e0, e1)); return r
    ctx.solve = timed
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); mg.plan(st, gl, env, seeds_ik); e1.record(); torch.cuda.synchronize()
    tot = e0.elapsed_time(e1)
    print("P", P, "total ms", round(tot, 2), [(tuple(s), round(a.elapsed_time(b), 2)) for s, a, b in log], flush=True)
    ctx.close()
