"""World-screen work counters (analysis tool, not the product path).

Builds a CRB_STATS=1 variant of the library next to this file (tools/libcurobo_stats.so, optionally
with the cuboid table forced to global memory, --gmem 1) and runs the bench workloads through it:
  [0] (group, cuboid) pairs examined, [1] pairs kept by the group-AABB culling,
  [2] pairs with an exact flag (some entry needs the slow path), [3] flagged entries (slow calls).
usage: python tools/world_stats.py [--mma 0|1]   (1: every environment on the GMEM build)
"""
import argparse
import ctypes as C
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--mma", type=int, default=1)
ap.add_argument("--problems", type=int, default=16)
ap.add_argument("--ftz", type=int, default=1, help="0: build without -ftz=true (A/B of the flag)")
args = ap.parse_args()

from paper_2310_17274_b200 import build as B  # noqa: E402

lib = os.path.join(ROOT, "tools", f"libcurobo_stats{args.mma}{'' if args.ftz else '_noftz'}.so")
if not os.path.exists(lib) or os.path.getmtime(lib) < max(os.path.getmtime(d) for d in B.DEPS):
    B.compile_lib(lib, ["-DCRB_STATS=1", "-DCRB_GMEM_MIN_K=0" if args.mma else "-DCRB_GMEM_MIN_K=100000"],
                  ftz=bool(args.ftz))
os.environ["CRB_LIB"] = lib

import torch  # noqa: E402
from paper_2310_17274_b200 import native, workload  # noqa: E402

so = C.CDLL(lib)
so.crb_debug_stats.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]


def stats(reset=True):
    a = (C.c_ulonglong * 32)()
    so.crb_debug_stats(a, int(reset))
    return list(a)


def run(name, wl):
    ctx = native.Context(0)
    ctx.set_robot(wl.robot); ctx.set_world(wl.worlds); ctx.set_cost_params(wl.cost)
    stats()
    kw = {"env": torch.tensor(wl.env, device="cuda")}
    if wl.start is not None:
        kw["start"] = torch.tensor(wl.start, device="cuda")
    ctx.solve(wl.solver, torch.tensor(wl.seeds, device="cuda"), torch.tensor(wl.goal, device="cuda"), **kw)
    s = stats()
    ctx.close()
    ex = max(s[0], 1)
    print(f"{name}: pairs {s[0]}  pre-screen-flagged {s[1] / ex:.3f}  exact-flagged {s[2] / ex:.3f}  "
          f"entries/pair {s[3] / ex:.3f}", flush=True)
    nd = max(s[14], 1)
    print(f"   sweep directions {s[14]}: with a hit sample {s[15] / nd:.3f}, segment bound skips {s[27] / nd:.3f} "
          f"(skips that would lose a hit: {s[28]}), samples per direction {s[26] / nd:.2f}", flush=True)
    wp = max(s[10], 1)
    print(f"   queue: world item {s[4] / max(s[8], 1):.0f} cyc x {s[8] / wp * 8:.1f}/pass, self item "
          f"{s[5] / max(s[9], 1):.0f} cyc x {s[9] / wp * 8:.1f}/pass; per warp-pass: in queue {s[7] / wp:.0f} cyc, "
          f"barrier wait {s[6] / wp:.0f} cyc", flush=True)
    fp = max(s[12], 1)
    print(f"   FK chain {s[11] / fp:.0f} cyc per pass, warp 0 waits {s[13] / fp:.0f} cyc at the placement barrier",
          flush=True)
    npass = max(s[25], 1)
    names = ["a2 state map", "FK chain + a8", "placement", "queue (pose, self, world)", "merge", "link sums",
             "joint grads", "transposed + gV"]
    ph = [s[16 + i] / npass for i in range(8)]
    tot = sum(ph)
    print("   phases (thread 0, cycles per pass): " + ", ".join(f"{n} {v:.0f} ({100 * v / tot:.1f}%)"
                                                              for n, v in zip(names, ph)) + f"; total {tot:.0f}",
          flush=True)


P = args.problems
run("cfg2 K=20 TO", workload.franka_to(0, list(range(P)), S=32, H=32, iters=100))
run("cfg3 K=20 IK", workload.franka_ik(0, list(range(300)), S=30, iters=100))
run("cfg5 K=1000 TO", workload.franka_to(0, list(range(4)), S=32, H=32, n_boxes=1000, iters=20, dense=True))
