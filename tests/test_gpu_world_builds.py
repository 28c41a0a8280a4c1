"""GPU: the two world builds and large worlds against the oracle.

The library builds its solver / evaluation kernels twice: <GMEM = true> reads the cuboid table from
global memory when some environment holds >= CRB_GMEM_MIN_K (60) enabled cuboids, else the table is
staged in shared memory.  The world arithmetic (culling, exact fp32 tests, accumulation order) is the
same, so on the SAME environments both builds return bitwise the same costs, gradients and solves;
a context whose world list includes one large environment runs the GMEM build for all of them.
Parity against the fp64 oracle at K in the GMEM range (ragged K, far and huge cuboids) uses the
tolerances of test_gpu_parity.py.
"""
import dataclasses

import numpy as np
import pytest
import torch

from paper_2310_17274_b200 import inputs, robots

from test_gpu_parity import ref_traj, MARGIN, Stats, T, f32, franka_trajs, make  # noqa: F401

pytestmark = pytest.mark.gpu

GMEM_MIN_K = 60


@pytest.fixture(scope="module")
def native():
    from paper_2310_17274_b200 import native as N
    return N


def _pair(native, rb, small, cp, big_k=80):
    """(shared-memory-table context over `small`, global-memory-table context over `small` + one big
    environment)."""
    big = inputs.random_world(9, 0, big_k, lo=-0.9, hi=0.9, disabled_frac=0.0)
    return make(native, rb, small, cp), make(native, rb, list(small) + [big], cp)


@pytest.mark.parametrize("flags", [inputs.SWEEP | inputs.SPEED, inputs.SPEED | inputs.JERK, 0])
def test_gmem_and_smem_builds_bitwise_equal_eval_to(native, O, flags):
    B, H = 48, 32
    rb, starts, goals_cfg, trajs = franka_trajs(70 + flags, B, H, noise=0.4)
    small = [inputs.tabletop_scene(1, e, 20) for e in range(2)] + [inputs.random_world(3, 0, 30, lo=-0.8, hi=0.8)]
    cp = inputs.CostParams(flags=flags, dt=0.25)
    smem, gmem = _pair(native, rb, small, cp)
    R = O.Robot(rb)
    goals = np.array([O.fk(R, q)[2] for q in goals_cfg])
    env = T((np.arange(B) % 3).astype(np.int32), torch.int32)
    a = smem.evaluate(T(f32(trajs)), T(f32(goals)), start=T(f32(starts)), env=env)
    b = gmem.evaluate(T(f32(trajs)), T(f32(goals)), start=T(f32(starts)), env=env)
    for x, y in zip(a, b):
        assert torch.equal(x, y)
    assert (a[2][:, 4] > 0).sum() >= B // 4          # the world term is active on many trajectories
    smem.close(); gmem.close()


def test_gmem_and_smem_builds_bitwise_equal_ik_and_solves(native, O):
    from paper_2310_17274_b200 import workload
    wl = workload.franka_to(0, list(range(4)), S=8, H=32, iters=15)
    smem, gmem = _pair(native, wl.robot, wl.worlds, wl.cost)
    outs = []
    for ctx in (smem, gmem):
        outs.append(ctx.solve(wl.solver, T(wl.seeds), T(wl.goal), start=T(wl.start), env=T(wl.env, torch.int32),
                              seed_outputs=True))
    for k in ("best_cost", "best_traj", "best_key", "seed_best_cost"):
        assert torch.equal(outs[0][k], outs[1][k]), k
    ik = workload.franka_ik(0, list(range(40)), S=30, iters=20)
    outs = []
    for ctx in (smem, gmem):
        ctx.set_cost_params(ik.cost)
        ctx.set_world(ik.worlds if ctx is smem else list(ik.worlds) + [inputs.random_world(9, 0, 80, disabled_frac=0.0)])
        outs.append(ctx.solve(ik.solver, T(ik.seeds), T(ik.goal), env=T(ik.env, torch.int32), seed_outputs=True))
    for k in ("best_cost", "best_traj", "seed_best_cost"):
        assert torch.equal(outs[0][k], outs[1][k]), k
    smem.close(); gmem.close()


@pytest.mark.parametrize("K,lo,hi,dmax", [(72, -0.8, 0.8, 0.3), (77, -0.7, 0.7, 0.25), (203, -0.9, 0.9, 0.12)])
def test_eval_to_parity_gmem_range(native, O, K, lo, hi, dmax):
    """Oracle parity with the GMEM build: K = 72, 77 (ragged last 32-cuboid culling block), 203 (~10 %
    disabled, so the enabled counts stay >= 64); rotated cuboids.  (Clutter and seed noise are
    sized so that sweep exits within the exclusion margin stay under the 2 % rule.)"""
    B, H = 128, 32
    rb, starts, goals_cfg, trajs = franka_trajs(300 + K, B, H, noise=0.3)
    worlds = [inputs.random_world(11, e, K, lo=lo, hi=hi, dmax=dmax) for e in range(2)]
    assert max(int(w.enabled.sum()) for w in worlds) >= GMEM_MIN_K     # the GMEM build runs
    cp = inputs.CostParams(flags=inputs.SWEEP | inputs.SPEED, dt=0.25)
    ctx = make(native, rb, worlds, cp)
    R = O.Robot(rb)
    Ws = [O.World(w) for w in worlds]
    env = (np.arange(B) % 2).astype(np.int32)
    goals = np.array([O.fk(R, q)[2] for q in goals_cfg])
    V, st, gl = f32(trajs), f32(starts), f32(goals)
    cost, grad, terms = ctx.evaluate(T(V), T(gl), start=T(st), env=T(env, torch.int32))
    cost, grad = cost.cpu().numpy(), grad.cpu().numpy()
    stats = Stats()
    active = 0
    for b in range(B):
        c_ref, g_ref, t_ref, margin = ref_traj(O, R, Ws[env[b]], cp, st[b], gl[b], V[b])
        stats.check(float(cost[b]), grad[b].astype(np.float64), c_ref, g_ref, margin, f"K={K} traj {b}")
        active += t_ref[4] > 0
    stats.done()
    assert active >= B // 4
    ctx.close()


def test_gmem_far_and_huge_cuboids(native, O):
    """Cuboids far outside the workspace (large offsets, still inside the fp16 range) and one
    beyond it (|offset| > 3e4 m: the pre-screen flags it and the exact test decides) next to a
    cuboid the arm penetrates: costs equal the FFMA build and the oracle."""
    B, H = 32, 32
    rb, starts, goals_cfg, trajs = franka_trajs(808, B, H, noise=0.3)
    base = inputs.random_world(12, 0, 70, lo=-0.8, hi=0.8, disabled_frac=0.0)
    pos = base.pos.copy(); dims = base.dims.copy()
    pos[3] = [2.0e3, -1.0e3, 5.0]                    # far, inside fp16 range
    pos[7] = [5.0e4, 0.0, 0.0]; dims[7] = [1.0, 1.0, 1.0]   # beyond the fp16 range
    pos[9] = [9.0e4, 0.0, 0.0]; dims[9] = [1.9e5, 2.0, 2.0]  # huge: contains the base of the arm
    pos[11] = [0.3, 0.0, 0.3]; dims[11] = [0.2, 0.2, 0.2]    # in the arm's way
    quat = base.quat.copy()
    quat[[7, 9]] = [1.0, 0.0, 0.0, 0.0]              # axis-aligned: the active faces stay exact in fp32
    w = inputs.World(pos, quat, dims, base.enabled)
    small = inputs.World(pos[:20].copy(), quat[:20].copy(), dims[:20].copy(), base.enabled[:20].copy())
    cp = inputs.CostParams(flags=inputs.SWEEP | inputs.SPEED, dt=0.25)
    R = O.Robot(rb)
    goals = np.array([O.fk(R, q)[2] for q in goals_cfg])
    V, st, gl = f32(trajs), f32(starts), f32(goals)
    ctx = make(native, rb, [w], cp)
    cost, grad, _ = ctx.evaluate(T(V), T(gl), start=T(st), env=T(np.zeros(B, np.int32), torch.int32))
    cost, grad = cost.cpu().numpy(), grad.cpu().numpy()
    Wo = O.World(w)
    stats = Stats()
    for b in range(B):
        c_ref, g_ref, t_ref, margin = ref_traj(O, R, Wo, cp, st[b], gl[b], V[b])
        stats.check(float(cost[b]), grad[b].astype(np.float64), c_ref, g_ref, margin, f"far {b}")
        assert t_ref[4] > 0                          # the huge cuboid contains the base spheres
    stats.done()
    # the 20-cuboid prefix through both builds: bitwise equal
    smem, gmem = _pair(native, rb, [small], cp)
    env = T(np.zeros(B, np.int32), torch.int32)
    a = smem.evaluate(T(V), T(gl), start=T(st), env=env)
    b2 = gmem.evaluate(T(V), T(gl), start=T(st), env=env)
    for x, y in zip(a, b2):
        assert torch.equal(x, y)
    ctx.close(); smem.close(); gmem.close()


def test_smem_build_far_and_huge_cuboids_against_oracle(native, O):
    """The small-world build (cuboid table in shared memory, K < 60) on cuboids far outside the workspace, one
    beyond the fp16 range (forced to the exact test), one huge cuboid containing the arm's base,
    and one in the arm's way: oracle parity."""
    B, H = 128, 32
    rb, starts, goals_cfg, trajs = franka_trajs(809, B, H, noise=0.3)
    base = inputs.random_world(13, 0, 24, lo=-0.8, hi=0.8, disabled_frac=0.0)
    pos = base.pos.copy(); dims = base.dims.copy(); quat = base.quat.copy()
    pos[3] = [2.0e3, -1.0e3, 5.0]
    pos[7] = [5.0e4, 0.0, 0.0]; dims[7] = [1.0, 1.0, 1.0]
    pos[9] = [9.0e4, 0.0, 0.0]; dims[9] = [1.9e5, 2.0, 2.0]
    pos[11] = [0.3, 0.0, 0.3]; dims[11] = [0.2, 0.2, 0.2]
    quat[[7, 9]] = [1.0, 0.0, 0.0, 0.0]
    w = inputs.World(pos, quat, dims, base.enabled)
    cp = inputs.CostParams(flags=inputs.SWEEP | inputs.SPEED, dt=0.25)
    R = O.Robot(rb)
    goals = np.array([O.fk(R, q)[2] for q in goals_cfg])
    V, st, gl = f32(trajs), f32(starts), f32(goals)
    ctx = make(native, rb, [w], cp)
    cost, grad, _ = ctx.evaluate(T(V), T(gl), start=T(st), env=T(np.zeros(B, np.int32), torch.int32))
    cost, grad = cost.cpu().numpy(), grad.cpu().numpy()
    Wo = O.World(w)
    stats = Stats()
    for b in range(B):
        c_ref, g_ref, t_ref, margin = ref_traj(O, R, Wo, cp, st[b], gl[b], V[b])
        stats.check(float(cost[b]), grad[b].astype(np.float64), c_ref, g_ref, margin, f"h2 far {b}")
        assert t_ref[4] > 0
    stats.done()        # deep inside the huge cuboid: many nearest-face ties (margin exclusions)
    ctx.close()


def _random_robot(seed, n_links=9, n_spheres=23):
    """A random tree (every Table 6 joint type, fixed links in the middle of the chain), an odd
    sphere count, 3 disabled spheres, a random pair list: the general paths of the kernels."""
    from test_oracle_kinematics import random_chain
    rb = random_chain(seed, n_links, n_spheres)
    g = np.random.default_rng(seed + 1)
    sph = rb.spheres.copy()
    sph[:, 3] = g.uniform(0.03, 0.09, n_spheres)
    sph[[2, 9, 17], 3] = -1.0                                    # disabled
    pairs = [(i, j) for i in range(n_spheres) for j in range(i + 1, n_spheres) if g.random() < 0.35]
    import dataclasses
    D = rb.n_dof
    return dataclasses.replace(rb, spheres=sph, pairs=np.array(pairs, np.int32), lo=-np.ones(D) * 2.5,
                               hi=np.ones(D) * 2.5, vmax=np.ones(D) * 2.0, amax=np.ones(D) * 15.0,
                               jmax=np.ones(D) * 500.0)


@pytest.mark.parametrize("seed,big", [(3, False), (4, False), (5, True)])
def test_random_robot_eval_parity_both_builds(native, O, seed, big):
    """Random robots (prismatic and revolute x/y/z joints, folded fixed links, 23 spheres of which
    3 disabled, random self pairs) through the TO and IK evaluations against the oracle, in the
    shared-memory-table build (K = 30) and the GMEM build (an extra 70-cuboid environment), plus an empty
    environment."""
    rb = _random_robot(seed)
    D, H, B = rb.n_dof, 16, 48
    g = np.random.default_rng(seed)
    worlds = [inputs.random_world(20 + seed, 0, 30, lo=-0.9, hi=0.9, dmax=0.3),
              inputs.World(np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0, 3)), np.zeros(0, np.int32))]
    if big:
        worlds.append(inputs.random_world(30 + seed, 0, 70, lo=-0.9, hi=0.9, dmax=0.2, disabled_frac=0.0))
    cp = inputs.CostParams(flags=inputs.SWEEP | inputs.SPEED | inputs.JERK, dt=0.1)
    ctx = make(native, rb, worlds, cp)
    R = O.Robot(rb)
    Ws = [O.World(w) for w in worlds]
    V = f32(g.uniform(-1.5, 1.5, (B, H, D)))
    st = f32(g.uniform(-1.0, 1.0, (B, D)))
    gl = f32(np.array([O.fk(R, g.uniform(-1, 1, D))[2] for _ in range(B)]))
    env = (np.arange(B) % len(worlds)).astype(np.int32)
    cost, grad, terms = ctx.evaluate(T(V), T(gl), start=T(st), env=T(env, torch.int32))
    cost, grad, terms = cost.cpu().numpy(), grad.cpu().numpy(), terms.cpu().numpy()
    stats = Stats()
    active_w = active_s = 0
    for b in range(B):
        c_ref, g_ref, t_ref, margin = ref_traj(O, R, Ws[env[b]], cp, st[b], gl[b], V[b])
        stats.check(float(cost[b]), grad[b].astype(np.float64), c_ref, g_ref, margin, f"rand TO {b}")
        active_w += t_ref[4] > 0
        active_s += t_ref[3] > 0
    stats.done()
    assert active_w >= 2 and active_s >= 2
    # IK mode (one configuration per row, all in the first environment)
    Q = f32(g.uniform(-1.5, 1.5, (40, D)))
    glq = f32(np.repeat(gl[:1], 40, 0))
    cq, gq, _ = ctx.evaluate(T(Q), T(glq), env=T(np.zeros(40, np.int32), torch.int32))
    cq, gq = cq.cpu().numpy(), gq.cpu().numpy()
    stats = Stats()
    for b in range(40):
        c_ref, g_ref, _, margin, _ = O.eval_ik(R, Ws[0], cp, glq[b], Q[b])
        stats.check(float(cq[b]), gq[b].astype(np.float64), c_ref, g_ref, ("ik", margin), f"rand IK {b}")
    stats.done()
    ctx.close()


def capacity_robot():
    """D = 16 joints on L = 32 links (every other link fixed, all revolute / prismatic types), 96
    spheres with a dense pair list (the capacity corner of the header)."""
    from test_oracle_kinematics import random_chain
    import dataclasses
    M = 96
    rb = random_chain(41, 32, M, types=[0, 4, 0, 5, 0, 6, 0, 1, 0, 4, 0, 2, 0, 5, 0, 3])
    D = rb.n_dof
    assert D == 16
    g = np.random.default_rng(42)
    sph = rb.spheres.copy()
    sph[:, 3] = g.uniform(0.02, 0.06, M)
    pairs = [(i, j) for i in range(M) for j in range(i + 1, M) if g.random() < 0.25]
    return dataclasses.replace(rb, spheres=sph, pairs=np.array(pairs, np.int32), lo=-np.ones(D) * 2.0,
                               hi=np.ones(D) * 2.0, vmax=np.ones(D) * 2.0, amax=np.ones(D) * 15.0,
                               jmax=np.ones(D) * 500.0)


@pytest.mark.parametrize("big", [False, True])
def test_capacity_robot_parity(native, O, big):
    """The capacity corner of the header: D = 16 joints on L = 32 links (every other link fixed,
    all revolute / prismatic types), H = 32 so H·D = 512, 96 spheres with a dense pair list.  TO
    and IK evaluations against the oracle in both world builds; short solves are bitwise
    repeatable and never worse than their seeds."""
    rb = capacity_robot()
    D, H, B = rb.n_dof, 32, 40
    g = np.random.default_rng(43)
    worlds = [inputs.random_world(61, 0, 24, lo=-1.2, hi=1.2, dmax=0.3)]
    if big:
        worlds.append(inputs.random_world(62, 0, 70, lo=-1.2, hi=1.2, dmax=0.2, disabled_frac=0.0))
    cp = inputs.CostParams(flags=inputs.SWEEP | inputs.SPEED | inputs.JERK, dt=0.1)
    ctx = make(native, rb, worlds, cp)
    n_cta, smem = ctx.solver_occupancy(H)
    assert n_cta >= 1 and smem <= 227 * 1024
    R = O.Robot(rb)
    Ws = [O.World(w) for w in worlds]
    st = f32(g.uniform(-1.0, 1.0, (B, D)))
    V = f32(np.clip(st[:, None, :] + np.cumsum(g.normal(0, 0.05, (B, H, D)), axis=1), -2.0, 2.0))
    gl = f32(np.array([O.fk(R, g.uniform(-1, 1, D))[2] for _ in range(B)]))
    env = (np.arange(B) % len(worlds)).astype(np.int32)
    cost, grad, _ = ctx.evaluate(T(V), T(gl), start=T(st), env=T(env, torch.int32))
    cost, grad = cost.cpu().numpy(), grad.cpu().numpy()
    stats = Stats()
    active_w = active_s = 0
    for b in range(B):
        c_ref, g_ref, t_ref, margin = ref_traj(O, R, Ws[env[b]], cp, st[b], gl[b], V[b])
        stats.check(float(cost[b]), grad[b].astype(np.float64), c_ref, g_ref, margin, f"cap TO {b}")
        active_w += t_ref[4] > 0
        active_s += t_ref[3] > 0
    stats.done()
    assert active_w >= 2 and active_s >= 2, (active_w, active_s)   # not vacuous
    Q = f32(g.uniform(-1.5, 1.5, (40, D)))
    glq = f32(np.repeat(gl[:1], 40, 0))
    cq, gq, _ = ctx.evaluate(T(Q), T(glq), env=T(np.zeros(40, np.int32), torch.int32))
    cq, gq = cq.cpu().numpy(), gq.cpu().numpy()
    stats = Stats()
    for b in range(40):
        c_ref, g_ref, _, margin, _ = O.eval_ik(R, Ws[0], cp, glq[b], Q[b])
        stats.check(float(cq[b]), gq[b].astype(np.float64), c_ref, g_ref, ("ik", margin), f"cap IK {b}")
    stats.done()
    sp = inputs.SolverParams(iters=8)
    seeds = V[:10].reshape(2, 5, H, D)
    runs = [ctx.solve(sp, T(seeds), T(gl[:2]), start=T(st[:2]), env=T(env[:2], torch.int32), seed_outputs=True)
            for _ in range(2)]
    for k in runs[0]:
        assert torch.equal(runs[0][k], runs[1][k]), k
    sbc = runs[0]["seed_best_cost"].cpu().numpy().reshape(-1)
    # seeds of problem p were evaluated above with env[p * 5 + s]; re-evaluate with the problem's env
    ce, _, _ = ctx.evaluate(T(V[:10]), T(np.repeat(gl[:2], 5, 0)), start=T(np.repeat(st[:2], 5, 0)),
                            env=T(np.repeat(env[:2], 5), torch.int32))
    assert np.all(sbc <= ce.cpu().numpy() * (1 + 1e-6))
    ik = ctx.solve(sp, T(f32(g.uniform(-1.5, 1.5, (2, 33, D)))), T(gl[:2]), env=T(env[:2], torch.int32),
                   seed_outputs=True)
    assert torch.isfinite(ik["seed_best_cost"]).all()
    ctx.close()


def test_capacity_d31_parity(native, O):
    """D = 31 (32 kinematic frames after folding, the subtree-mask limit) on 36 links with all
    Table 6 joint types, 40 spheres: TO evaluation at H = 16 (H*D = 496 <= 512) and IK evaluation
    against the oracle; D = 32 is refused with CRB_E_LIMIT."""
    from test_oracle_kinematics import random_chain
    import dataclasses
    types = [0] + [4, 5, 6, 1, 2, 3, 4, 0] * 5
    types = types[:36]
    rb = random_chain(77, 36, 40, types=types)
    D = rb.n_dof
    assert D == 31, D
    g = np.random.default_rng(78)
    sph = rb.spheres.copy()
    sph[:, 3] = g.uniform(0.02, 0.05, 40)
    pairs = [(i, j) for i in range(40) for j in range(i + 1, 40) if g.random() < 0.3]
    rb = dataclasses.replace(rb, spheres=sph, pairs=np.array(pairs, np.int32), lo=-np.ones(D) * 1.5,
                             hi=np.ones(D) * 1.5, vmax=np.ones(D) * 2.0, amax=np.ones(D) * 15.0, jmax=np.ones(D) * 500.0)
    worlds = [inputs.random_world(63, 0, 24, lo=-1.5, hi=1.5, dmax=0.3)]
    cp = inputs.CostParams(flags=inputs.SWEEP | inputs.SPEED | inputs.JERK, dt=0.1)
    ctx = make(native, rb, worlds, cp)
    R, W = O.Robot(rb), O.World(worlds[0])
    H, B = 16, 24
    st = f32(g.uniform(-0.5, 0.5, (B, D)))
    V = f32(np.clip(st[:, None, :] + np.cumsum(g.normal(0, 0.03, (B, H, D)), axis=1), -1.5, 1.5))
    gl = f32(np.array([O.fk(R, g.uniform(-0.5, 0.5, D))[2] for _ in range(B)]))
    cost, grad, _ = ctx.evaluate(T(V), T(gl), start=T(st), env=T(np.zeros(B, np.int32), torch.int32))
    cost, grad = cost.cpu().numpy(), grad.cpu().numpy()
    stats = Stats()
    for b in range(B):
        c_ref, g_ref, t_ref, margin = ref_traj(O, R, W, cp, st[b], gl[b], V[b])
        stats.check(float(cost[b]), grad[b].astype(np.float64), c_ref, g_ref, margin, f"d31 TO {b}")
    stats.done()
    Q = f32(g.uniform(-1.0, 1.0, (40, D)))
    glq = f32(np.repeat(gl[:1], 40, 0))
    cq, gq, _ = ctx.evaluate(T(Q), T(glq), env=T(np.zeros(40, np.int32), torch.int32))
    cq, gq = cq.cpu().numpy(), gq.cpu().numpy()
    stats = Stats()
    for b in range(40):
        c_ref, g_ref, _, margin, _ = O.eval_ik(R, W, cp, glq[b], Q[b])
        stats.check(float(cq[b]), gq[b].astype(np.float64), c_ref, g_ref, ("ik", margin), f"d31 IK {b}")
    stats.done()
    # short solves run (TO and IK with the particle warm-up: D * 32 = 992 elements per group)
    out = ctx.solve(inputs.SolverParams(iters=5), T(V.reshape(2, 12, H, D)), T(gl[:2]), start=T(st[:2]), seed_outputs=True)
    assert torch.isfinite(out["seed_best_cost"]).all()
    ik = ctx.solve(inputs.SolverParams(iters=5, particle_iters=2, n_particles=8), T(Q.reshape(2, 20, D)), T(gl[:2]),
                   seed_outputs=True)
    assert torch.isfinite(ik["seed_best_cost"]).all()
    # the persistent schedules at D = 31 (the IK step's 32-register bucket, 992-element groups in the
    # saved state) against one CTA per group / seed, bitwise
    for sp in (inputs.SolverParams(iters=6, persist=3), inputs.SolverParams(iters=6, particle_iters=1, n_particles=8,
                                                                             persist=2)):
        ik_p = ctx.solve(sp, T(Q.reshape(2, 20, D)), T(gl[:2]), seed_outputs=True)
        ik_0 = ctx.solve(dataclasses.replace(sp, persist=0), T(Q.reshape(2, 20, D)), T(gl[:2]), seed_outputs=True)
        to_p = ctx.solve(sp, T(V.reshape(2, 12, H, D)), T(gl[:2]), start=T(st[:2]), seed_outputs=True)
        to_0 = ctx.solve(dataclasses.replace(sp, persist=0), T(V.reshape(2, 12, H, D)), T(gl[:2]), start=T(st[:2]),
                         seed_outputs=True)
        for k in ik_p:
            assert torch.equal(ik_p[k], ik_0[k]), ("IK", k)
            assert torch.equal(to_p[k], to_0[k]), ("TO", k)
    ctx.close()
    big = random_chain(79, 40, 10, types=[0] + [4] * 39)
    assert big.n_dof == 39
    c2 = native.Context(0)
    with pytest.raises(native.CrbError) as e:
        c2.set_robot(big)
    assert e.value.code == -6
    c2.close()


def test_set_world_rejects_more_than_max_cuboids(native):
    """crb_set_world: k_max above CRB_MAX_CUBOIDS (131071; the large-world slow path packs the
    cuboid index in 17 bits) returns CRB_E_SHAPE before reading any cuboid."""
    import ctypes as C
    ctx = native.Context(0)
    counts = (C.c_int * 1)(0)
    arr = (native.crb_cuboid * 1)()
    rc = native._lib.crb_set_world(ctx.h, 1, 131072, counts, arr)
    assert rc == -2                                    # CRB_E_SHAPE
    assert native._lib.crb_set_world(ctx.h, 1, 131071, counts, arr) == 0
    ctx.close()
