"""One cfg-3 IK solve (for ncu) or a short timing: P goals x 30 seeds x 100 iterations, shared K = 20 scene.
usage: python tools/prof_ik.py [P=1000] [cluster=-1 (auto) | 0 | 1] [reps=1] [persist=-1]"""
import dataclasses, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_17274_b200 import native, workload
P = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
cl = int(sys.argv[2]) if len(sys.argv) > 2 else -1
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
pe = int(sys.argv[4]) if len(sys.argv) > 4 else -1
wl = workload.franka_ik(0, list(range(P)), S=30, iters=100)
ctx = native.Context(0)
ctx.set_robot(wl.robot); ctx.set_world(wl.worlds); ctx.set_cost_params(wl.cost)
sp = dataclasses.replace(wl.solver, cluster=cl, persist=pe)
args = (torch.tensor(wl.seeds, device="cuda"), torch.tensor(wl.goal, device="cuda"))
kw = dict(env=torch.tensor(wl.env, device="cuda"))
ctx.solve(sp, *args, **kw)
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); ctx.solve(sp, *args, **kw); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = sorted(ts)[len(ts) // 2]
lib = os.path.basename(os.environ.get("CRB_LIB", "in-tree"))
print(f"IK {lib} P={P} cluster={cl} persist={pe}: {ms:.2f} ms (median of {reps}), {P / (ms * 1e-3):.0f} queries/s")
