"""Persistent-schedule chunk-count sweep (analysis tool): solve time of the bench workloads for
several iteration-chunk counts (SolverParams.persist = k).  usage: python tools/chunk_sweep.py"""
import dataclasses, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_17274_b200 import native, workload


def timed(ctx, sp, args, kw, reps=5):
    ctx.solve(sp, *args, **kw); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); ctx.solve(sp, *args, **kw); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def sweep(name, wl, ks, to=True):
    ctx = native.Context(0)
    ctx.set_robot(wl.robot); ctx.set_world(wl.worlds); ctx.set_cost_params(wl.cost)
    args = (torch.tensor(wl.seeds, device="cuda"), torch.tensor(wl.goal, device="cuda"))
    kw = dict(env=torch.tensor(wl.env, device="cuda"))
    if to:
        kw["start"] = torch.tensor(wl.start, device="cuda")
    res = {k: round(timed(ctx, dataclasses.replace(wl.solver, persist=k), args, kw), 3) for k in ks}
    print(name, res, flush=True)
    ctx.close()


sweep("cfg2 ms", workload.franka_to(0, list(range(64)), S=32, H=32, iters=100), [6, 8, 10, 12, 14, 16, 20])
sweep("cfg4 ms", workload.franka_to(0, list(range(128)), S=12, H=32, iters=100), [6, 8, 10, 12, 14, 16, 20])
sweep("cfg5(64 problems) ms", workload.franka_to(0, list(range(64)), S=32, H=32, n_boxes=1000, iters=100, dense=True),
      [5, 10, 16, 20, 25])
sweep("cfg3 IK ms", workload.franka_ik(0, list(range(1000)), S=30, iters=100), [8, 12, 16, 20, 25, 32], to=False)
