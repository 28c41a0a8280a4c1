"""IK throughput, sequential vs cluster latency mode (analysis tool for the automatic rule)."""
import os, sys, dataclasses
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_17274_b200 import native, workload
def timeit(ctx, sp, args, kw, n=3):
    ctx.solve(sp, *args, **kw); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): ctx.solve(sp, *args, **kw)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
for P, parts in [(1000, 0), (1000, 2), (300, 0), (150, 0), (64, 2)]:
    wl = workload.franka_ik(0, list(range(P)), S=30, iters=100)
    ctx = native.Context(0); ctx.set_robot(wl.robot); ctx.set_world(wl.worlds); ctx.set_cost_params(wl.cost)
    args = (torch.tensor(wl.seeds, device="cuda"), torch.tensor(wl.goal, device="cuda"))
    kw = dict(env=torch.tensor(wl.env, device="cuda"))
    sp = dataclasses.replace(wl.solver, particle_iters=parts)
    r = {c: round(timeit(ctx, dataclasses.replace(sp, cluster=c), args, kw), 2) for c in (0, 1, -1)}
    print(f"IK P={P} particles={parts}: seq {r[0]} ms, cluster {r[1]} ms, auto {r[-1]} ms", flush=True)
    ctx.close()
