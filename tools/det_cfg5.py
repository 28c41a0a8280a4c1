"""Determinism probe (analysis tool): the same cfg-5 (dense K = 1000) solve several times, outputs compared
bitwise.  usage: python tools/det_cfg5.py [P=64] [iters=10] [reps=3]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_17274_b200 import native, workload
P = int(sys.argv[1]) if len(sys.argv) > 1 else 64
it = int(sys.argv[2]) if len(sys.argv) > 2 else 10
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
wl = workload.franka_to(0, list(range(P)), S=32, H=32, n_boxes=1000, iters=it, dense=True)
ctx = native.Context(0)
ctx.set_robot(wl.robot); ctx.set_world(wl.worlds); ctx.set_cost_params(wl.cost)
args = (wl.solver, torch.tensor(wl.seeds, device="cuda"), torch.tensor(wl.goal, device="cuda"))
kw = dict(start=torch.tensor(wl.start, device="cuda"), env=torch.tensor(wl.env, device="cuda"), seed_outputs=True)
outs = []
for r in range(reps):
    o = ctx.solve(*args, **kw); torch.cuda.synchronize()
    outs.append([t.clone() if torch.is_tensor(t) else t for t in (o if isinstance(o, (list, tuple)) else o.values())])
same = all(all(torch.equal(a, b) for a, b in zip(outs[0], o) if torch.is_tensor(a)) for o in outs[1:])
print(f"P={P} iters={it} reps={reps}: bitwise identical across runs: {same}")
