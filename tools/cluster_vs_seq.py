import sys, dataclasses
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2310_17274_b200 import native, workload
def timeit(ctx, sp, args, kw, n=3):
    ctx.solve(sp, *args, **kw); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): ctx.solve(sp, *args, **kw)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
for (P, S, parts) in [(64, 12, 2), (32, 12, 2), (32, 12, 0), (16, 32, 0), (12, 32, 0), (24, 12, 0)]:
    wl = workload.franka_to(0, list(range(P)), S=S, H=32, iters=100)
    ctx = native.Context(0); ctx.set_robot(wl.robot); ctx.set_world(wl.worlds); ctx.set_cost_params(wl.cost)
    args = (torch.tensor(wl.seeds, device="cuda"), torch.tensor(wl.goal, device="cuda"))
    kw = dict(start=torch.tensor(wl.start, device="cuda"), env=torch.tensor(wl.env, device="cuda"))
    sp = dataclasses.replace(wl.solver, particle_iters=parts)
    r = {c: round(timeit(ctx, dataclasses.replace(sp, cluster=c), args, kw), 2) for c in (0, 1)}
    print(f"P={P} S={S} particles={parts}: seq {r[0]} ms, cluster {r[1]} ms", flush=True)
    ctx.close()
