"""One cfg-5 TO solve (for ncu): dense K = 1000 world, P problems x 32 seeds x 32 timesteps x iters.
usage: python tools/prof_cfg5.py [P=16] [iters=30]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_17274_b200 import native, workload
P = int(sys.argv[1]) if len(sys.argv) > 1 else 16
it = int(sys.argv[2]) if len(sys.argv) > 2 else 30
wl = workload.franka_to(0, list(range(P)), S=32, H=32, n_boxes=1000, iters=it, dense=True)
ctx = native.Context(0)
ctx.set_robot(wl.robot); ctx.set_world(wl.worlds); ctx.set_cost_params(wl.cost)
args = (wl.solver, torch.tensor(wl.seeds, device="cuda"), torch.tensor(wl.goal, device="cuda"))
kw = dict(start=torch.tensor(wl.start, device="cuda"), env=torch.tensor(wl.env, device="cuda"))
ctx.solve(*args, **kw); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); ctx.solve(*args, **kw); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"cfg5 P={P} iters={it}: {ms:.2f} ms, {wl.evals_per_solve() / (ms * 1e-3) / 1e6:.2f} M evals/s")
