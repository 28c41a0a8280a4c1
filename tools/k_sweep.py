"""Solve time vs cuboid count for the library at CRB_LIB (analysis tool): tabletop scenes with K
cuboids (table + K-1 boxes), 32 problems x 32 seeds x 32 timesteps x 30 iterations."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_17274_b200 import native, workload

out = {}
for K in [int(k) for k in (sys.argv[1] if len(sys.argv) > 1 else "20,32,48,64,96,128").split(",")]:
    wl = workload.franka_to(0, list(range(32)), S=32, H=32, n_boxes=K, iters=30)
    ctx = native.Context(0)
    ctx.set_robot(wl.robot); ctx.set_world(wl.worlds); ctx.set_cost_params(wl.cost)
    args = (wl.solver, torch.tensor(wl.seeds, device="cuda"), torch.tensor(wl.goal, device="cuda"))
    kw = dict(start=torch.tensor(wl.start, device="cuda"), env=torch.tensor(wl.env, device="cuda"))
    ctx.solve(*args, **kw); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        ctx.solve(*args, **kw)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    out[K] = round(wl.evals_per_solve() / (ms * 1e-3) / 1e6, 1)
    ctx.close()
print(os.environ.get("CRB_LIB", "default"), json.dumps(out))
if len(sys.argv) > 2 and sys.argv[2] == "dense":
    wl = workload.franka_to(0, list(range(16)), S=32, H=32, n_boxes=1000, iters=30, dense=True)
    ctx = native.Context(0)
    ctx.set_robot(wl.robot); ctx.set_world(wl.worlds); ctx.set_cost_params(wl.cost)
    args = (wl.solver, torch.tensor(wl.seeds, device="cuda"), torch.tensor(wl.goal, device="cuda"))
    kw = dict(start=torch.tensor(wl.start, device="cuda"), env=torch.tensor(wl.env, device="cuda"))
    ctx.solve(*args, **kw); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); ctx.solve(*args, **kw); e1.record(); torch.cuda.synchronize()
    print("dense1000", round(wl.evals_per_solve() / (e0.elapsed_time(e1) * 1e-3) / 1e6, 2), "M evals/s")
