"""Randomised parity stress (analysis tool, GPU): random robots (every joint type, 4-13 links, 6-59
spheres, random self pairs), random worlds (K = 3..149, so both world builds), random trajectories
(H = 8..64, so the timestep windows) and IK batches; GPU costs against the fp64 oracle.  Reports the
evaluations whose cost differs by more than 1e-4 relative (floor 0.1) outside the oracle's branch
margins.  usage: python tools/stress_parity.py [end_case=40] [start_case=0]
Round 2: cases 0..259, 16,640 evaluations: one outlier, an IK pose term at 2.4e-4 relative (the
rotation error 1 - |<q_g, q>| of a 13-link random chain, fp32 forward-kinematics error), no world or
self-collision mismatch."""
import os, sys, dataclasses
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
from oracle import oracle as O
from paper_2310_17274_b200 import inputs, native
from test_oracle_kinematics import random_chain
T = lambda a, dt=torch.float32: torch.tensor(np.ascontiguousarray(a), dtype=dt, device="cuda")
f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)
bad = 0; total = 0; skipped = 0; worst = 0.0
for case in range(int(sys.argv[2]) if len(sys.argv) > 2 else 0, int(sys.argv[1]) if len(sys.argv) > 1 else 40):
    g = np.random.default_rng(1000 + case)
    nl = int(g.integers(4, 14)); ns = int(g.integers(6, 60))
    rb = random_chain(5000 + case, nl, ns)
    D = rb.n_dof
    M = ns
    pairs = [(i, j) for i in range(M) for j in range(i + 1, M) if g.random() < 0.4]
    if not pairs: pairs = [(0, 1)]
    rb = dataclasses.replace(rb, pairs=np.array(pairs, np.int32), vmax=np.ones(D) * 3.0, amax=np.ones(D) * 30.0,
                             jmax=np.ones(D) * 500.0)
    K = int(g.integers(3, 150))
    worlds = [inputs.random_world(case, e, K, lo=-1.2, hi=1.2, dmax=float(g.uniform(0.1, 0.6))) for e in range(2)]
    flags = int(g.integers(0, 8)) & 7
    H = int(g.choice([8, 12, 16, 24, 32, 40, 50, 64]))
    if H * D > 512: H = max(8, 512 // D)
    cp = inputs.CostParams(flags=flags, dt=0.1)
    try:
        ctx = native.Context(0); ctx.set_robot(rb); ctx.set_world(worlds); ctx.set_cost_params(cp)
    except native.CrbError as e:
        print("skip robot", case, e); continue
    R = O.Robot(rb); Ws = [O.World(w) for w in worlds]
    B = 24
    st = f32(g.uniform(-1.0, 1.0, (B, D)))
    V = f32(np.clip(st[:, None, :] + np.cumsum(g.normal(0, float(g.uniform(0.01, 0.2)), (B, H, D)), axis=1), -3, 3))
    gl = f32(np.array([O.fk(R, g.uniform(-1, 1, D))[2] for _ in range(B)]))
    env = (np.arange(B) % 2).astype(np.int32)
    cost, grad, terms = ctx.evaluate(T(V), T(gl), start=T(st), env=T(env, torch.int32))
    cost, terms = cost.cpu().numpy(), terms.cpu().numpy()
    for b in range(B):
        c, gr, t, _, _, sm, cm = O.eval_traj(R, Ws[env[b]], cp, st[b], gl[b], V[b], state_margins=True)
        total += 1
        if cm < 2e-5 or np.min(sm) < 2e-5: skipped += 1; continue
        err = abs(cost[b] - c) / (abs(c) + 1e-1)
        worst = max(worst, err)
        if err > 1e-4:
            bad += 1
            print(f"case {case} K={K} H={H} D={D} flags={flags} b={b}: gpu {cost[b]:.6g} ref {c:.6g} terms gpu {terms[b]} ref {np.asarray(t)}")
    # IK evaluation
    Q = f32(g.uniform(-3, 3, (40, D)))
    glq = f32(np.repeat(gl[:1], 40, 0))
    cq, _, tq = ctx.evaluate(T(Q), T(glq), env=T(np.zeros(40, np.int32), torch.int32))
    cq = cq.cpu().numpy()
    for b in range(40):
        c, gr, t, m, _ = O.eval_ik(R, Ws[0], cp, glq[b], Q[b])
        total += 1
        if m < 2e-5: skipped += 1; continue
        err = abs(cq[b] - c) / (abs(c) + 1e-1)
        worst = max(worst, err)
        if err > 1e-4:
            bad += 1; print(f"IK case {case} K={K} D={D} b={b}: gpu {cq[b]:.6g} ref {c:.6g}")
    ctx.close()
print(f"total {total} skipped(margin) {skipped} bad {bad} worst rel err {worst:.3g}")
