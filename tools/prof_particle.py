"""Particle warm-up (f1) timing / profiling driver: cfg2 workload, iters = 0, 2 x 64 particles.
usage: python tools/prof_particle.py [P] [sigma0_frac ...]   (ncu: -k regex:solve_to -c 1)"""
import dataclasses
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2310_17274_b200 import native, workload  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 10
fracs = [float(a) for a in sys.argv[2:]] or [0.1]
dev = torch.device("cuda:0")
wl = workload.franka_to(0, list(range(P)), S=32, H=32, iters=100)
ctx = native.Context(0)
ctx.set_robot(wl.robot); ctx.set_world(wl.worlds); ctx.set_cost_params(wl.cost)
a = (torch.tensor(wl.seeds, device=dev), torch.tensor(wl.goal, device=dev))
kw = dict(start=torch.tensor(wl.start, device=dev), env=torch.tensor(wl.env, device=dev))
for fr in fracs:
    for iters, pit in [(0, 2), (25, 0)]:
        sp = dataclasses.replace(wl.solver, iters=iters, particle_iters=pit, n_particles=64, sigma0_frac=fr)
        ctx.solve(sp, *a, **kw)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); ctx.solve(sp, *a, **kw); e1.record(); torch.cuda.synchronize()
        passes = pit * 64 + 1 + iters * 4
        print(f"sigma0_frac={fr} iters={iters} particle_iters={pit}: {e0.elapsed_time(e1):.2f} ms, "
              f"{e0.elapsed_time(e1) / passes * 1e3:.1f} us/pass")
