"""cfg2-style TO solve timing for a given schedule (analysis tool): P problems x S seeds x 32 x iters.
usage: python tools/prof_to.py [P=64] [S=32] [persist=-1] [reps=5]"""
import dataclasses, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_17274_b200 import native, workload
P = int(sys.argv[1]) if len(sys.argv) > 1 else 64
S = int(sys.argv[2]) if len(sys.argv) > 2 else 32
pe = int(sys.argv[3]) if len(sys.argv) > 3 else -1
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
wl = workload.franka_to(0, list(range(P)), S=S, H=32, iters=100)
ctx = native.Context(0)
ctx.set_robot(wl.robot); ctx.set_world(wl.worlds); ctx.set_cost_params(wl.cost)
sp = dataclasses.replace(wl.solver, persist=pe, cluster=0)
args = (sp, torch.tensor(wl.seeds, device="cuda"), torch.tensor(wl.goal, device="cuda"))
kw = dict(start=torch.tensor(wl.start, device="cuda"), env=torch.tensor(wl.env, device="cuda"))
ctx.solve(*args, **kw); torch.cuda.synchronize()
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); ctx.solve(*args, **kw); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = sorted(ts)[len(ts) // 2]
print(f"TO P={P} S={S} persist={pe}: {ms:.2f} ms, {wl.evals_per_solve() / (ms * 1e-3) / 1e6:.1f} M evals/s")
